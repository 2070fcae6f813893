// Internal shared pieces of libkp: status plumbing, launch argument block,
// and the async-copy PTX wrappers every family uses.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <string>

#include "../../include/kp_abi.h"

namespace kp {

// Set the thread-local last-error message and return `st`.
kp_status fail(kp_status st, const std::string& msg);
// Count launches issued through the library (kp_launch_count()).
void note_launch(int64_t n = 1);
// Check the last launch; maps a CUDA error to KP_ERR_CUDA with a message.
kp_status check_launch(const char* what);

// One GEMM problem as every family's launcher sees it (validated).
struct GemmProblem {
    int64_t batch, m, n, k;
    bool ta, tb;
    int64_t lda, ldb, ldc;
    int64_t sa, sb, sc;
    float alpha, beta;
    const void* A;
    const void* B;
    float* C;
};

// Ordered stream-K hand-off flags: a per-device ring of KP_SK_RING u32 slots
// (allocated and zeroed once, the only device memory the library owns).  Each
// stream-K launch reserves gridDim.x consecutive slots and a fresh epoch, so
// concurrent or back-to-back launches never read each other's flags.
constexpr uint32_t KP_SK_RING = 1u << 16;
constexpr uint32_t KP_SK_RING_MASK = KP_SK_RING - 1;
struct SkFlags {
    uint32_t* flags;
    uint32_t base, epoch;
};
// Reserve `n` slots on the current device (KP_ERR_CUDA if the ring cannot be
// allocated).
kp_status sk_reserve(uint32_t n, SkFlags* out);
// Scheduling policy of the K1 family: 0 = one tile per CTA, 1 = ordered
// stream-K when the last wave would leave SMs idle (default), 2 = ordered
// stream-K whenever the problem has at least two tiles (tests).
int simt_schedule();
// Number of SMs of the current device (cached).
int sm_count();
// The calling thread's current CUDA device (0 if the query fails).
inline int current_device() {
    int dev = 0;
    return cudaGetDevice(&dev) == cudaSuccess ? dev : 0;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ---------------------------------------------------------------- PTX ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 16-byte global->shared async copy to a shared-window address; bytes beyond
// `src_bytes` are zero-filled (src_bytes 0 reads nothing, so `src` may then
// point anywhere).
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n"
                 :: "r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
// Full 16-byte copy (interior tiles: no zero-fill operand).
__device__ __forceinline__ void cp_async16_full(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" :: "r"(dst), "l"(src) : "memory");
}
// 4-byte variant (unaligned rows, transposes, tails); src_bytes 0 writes a zero.
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, int src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n"
                 :: "r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async4_full(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" :: "r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" :: "n"(N) : "memory");
}

}  // namespace kp
