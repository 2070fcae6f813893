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
// 4-byte variant (unaligned rows, transposes, tails); src_bytes 0 writes a zero.
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, int src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n"
                 :: "r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" :: "n"(N) : "memory");
}

}  // namespace kp
