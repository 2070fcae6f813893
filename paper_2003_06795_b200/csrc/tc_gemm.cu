// K2 / K3: tcgen05 tensor-core GEMM families (TF32 and BF16 inputs, FP32
// accumulate in TMEM, FP32 output), same C = alpha*op(A)@op(B) + beta*C
// contract and operand layouts as K1.
//
// Kernel anatomy (one 128 x BN output tile per CTA, 6 warps):
//   warp 0  TMA producer: per stage one K slice of 128 bytes per row
//           (32 tf32 / 64 bf16), A 128 x 128 B and B BN x 128 B, SWIZZLE_128B,
//           zero fill for M/N/K tails, 3-D maps so batches never bleed;
//   warp 1  TMEM allocator + single-thread tcgen05.mma issuer
//           (M=128, N=BN, K=8 tf32 / 16 bf16 per instruction), tcgen05.commit
//           releases the stage and finally signals the epilogue;
//   warps 2-5 epilogue: tcgen05.ld 32x32b.x32 of their TMEM lane quarter,
//           transpose through padded shared memory, coalesced fp32 stores
//           with alpha/beta and bounds checks.
// K-major operands (A normal, B transposed) and MN-major operands (A
// transposed, B normal) differ only in the TMA box and the UMMA descriptor
// (K-major: rows of 128 B, SBO 1024; MN-major: 128-byte MN atoms of 8 K rows,
// LBO = BK*128, SBO = 1024), so all four layouts run without a transpose.
//
// Config encoding into the reference's 5-field KernelConfig:
//   col_tile 1,2,4,8  -> BN = 32, 64, 128, 256 (UMMA N, TMEM columns)
//   acc      1,2,4,8  -> pipeline stages 2, 3, 4, 6 (clamped to shared memory)
//   row_tile 1        -> BM = 128 (cta_group::1)
//   wg       (8, 8)   -> one tile per CTA, grouped raster
//   wg     (16, 16)   -> persistent CTAs (grid = SM count), double-buffered
//                        TMEM accumulator: epilogue of tile i overlaps the
//                        MMAs of tile i+1
//   row_tile 2        -> CTA pair, cta_group::2, M = 256 (persistent, ct 4|8)
// 40 configs per family, canonical KernelConfig order.
//
// Split-K (1-CTA kernels, kp_set_tc_split): when the output tiles fill less
// than half of the SMs -- deep-K network GEMMs such as ResNet-50 c5_3x3 at
// batch 8 (392 x 4608 x 512: 16 tiles of 128 x 128 on 148 SMs) -- each tile's
// K range is cut into S contiguous k-tile ranges, one work unit each, and
// every unit writes its fp32 partial tile to a per-device workspace. A second
// kernel (tc_splitk_reduce, launched with programmatic dependent launch so its
// launch overlaps the GEMM) sums the S partials of every element in split
// order 0..S-1 -- fixed, so results are run-to-run deterministic -- applies
// alpha / beta and writes C. (Reducing in the last-arriving unit instead
// serialises S x 64-128 KB of L2 reads through one SM per tile: measured 2x
// slower than no split at all on c5_3x3.)
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "tc_registry.h"

namespace kp {
namespace tc {

constexpr int BM = 128;
constexpr int NUM_THREADS = 192;
constexpr int GROUP_M = 8;  // default raster group (tc_group_m())
constexpr int STAGE_ALIGN = 1024;
constexpr int EPI_PITCH = 33;  // padded 32x32 staging tile per epilogue warp (fallback path)
// Epilogue shared memory: per epilogue warp two 32x32 fp32 buffers (4 KB,
// 128B-swizzled rows) for the TMA-store path; the fallback path's padded
// staging tiles fit in the same 32 KB.
constexpr int EPI_BUF = 32 * 32 * 4;
constexpr int EPI_BYTES = 4 * 2 * EPI_BUF;

struct TcParams {
    float* C;
    int M, N, K;
    int64_t ldc, sc;
    float alpha, beta;
    int tiles_m, tiles_n;
    int stages, k_tiles;
    int batch;
    int a_batch, b_batch;  // 1 if the operand advances with the batch index, else 0
    int splits;            // K splits per tile (1 = no split-K)
    int group_m;           // m-tiles per raster group
    int tma_store;         // 1: C tile stored by TMA (beta == 0, aligned C, no split-K);
                           // 2: split-K partial tiles stored by TMA into the workspace
    float* ws;             // split-K partial tiles [tile][split][BM][BN] (splits > 1)
};

// k-tile range [kb0, kb1) of split s of S over k_tiles (never empty for S <= k_tiles)
__device__ __forceinline__ void split_range(int s, int S, int k_tiles, int& kb0, int& kb1) {
    kb0 = int((int64_t(s) * k_tiles) / S);
    kb1 = int((int64_t(s + 1) * k_tiles) / S);
}

// ------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    return ok != 0;
}
// Wait for the phase of parity `parity`; a watchdog (~2^34 cycles, ~8 s)
// turns a pipeline deadlock into a trapped launch error instead of a hung GPU.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    if (mbar_try(bar, parity)) return;
    const long long t0 = clock64();
    while (!mbar_try(bar, parity)) {
        if (clock64() - t0 > (1LL << 34)) {
#ifdef KP_TC_DEBUG
            printf("tc watchdog: block (%d,%d) thread %d bar 0x%x parity %u\n", blockIdx.x,
                   blockIdx.z, threadIdx.x, bar, parity);
#endif
            __trap();
        }
    }
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];"
        :: "r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(bar) : "memory");
}
__device__ __forceinline__ void fence_after_sync() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_before_sync() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

// KP_TC_DEBUG builds (libkp_debug.so) record per-CTA phase timestamps
// (%globaltimer, ns) of the 1-CTA kernel for the first TRACE_CTAS CTAs of a
// launch: 0 entry, 1 setup done, 2 first TMA issued, 3 first stage landed,
// 4 last MMA issued, 5 accumulator complete (epilogue), 6 stores issued,
// 7 exit; 8.. epilogue warp 2, TMA-store path: chunk c's TMEM data in
// registers (8 + 2c) and its store issued (9 + 2c), first 4 chunks.
// kp_tc_trace_dump() copies them out (tools/tc_trace.py).
#ifdef KP_TC_DEBUG
constexpr int TRACE_CTAS = 4096;
__device__ unsigned long long g_tc_trace[TRACE_CTAS][16];
__device__ __forceinline__ void trace(int slot) {
    if (blockIdx.x < TRACE_CTAS) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_tc_trace[blockIdx.x][slot] = t;
    }
}
#else
__device__ __forceinline__ void trace(int) {}
#endif

// UMMA shared-memory descriptor (Blackwell version bits = 1). layout: 2 =
// SWIZZLE_128B, 4 = SWIZZLE_64B, 1 = SWIZZLE_128B_BASE32B.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
    uint64_t d = 0;
    d |= uint64_t((addr >> 4) & 0x3FFF);
    d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
    d |= uint64_t(1) << 46;  // descriptor version (sm_100)
    d |= uint64_t(layout & 7) << 61;
    return d;
}

// Shared layout of an MN-major operand tile (MN contiguous in global memory):
// atoms W bytes wide along MN, one K row per W bytes, GROUP K rows per
// swizzle group. TF32 must use the 32-byte-granular 128B swizzle (UMMA
// SWIZZLE_128B_BASE32B, TMA SWIZZLE_128B_ATOM_32B); BF16 uses SWIZZLE_128B,
// or SWIZZLE_64B when the tile is only 32 elements wide.
template <int ES, int EXTENT>
struct MnMajor {
    static constexpr int W = (ES == 2 && EXTENT < 64) ? 64 : 128;  // bytes per atom row
    static constexpr int ATOM = W / ES;                             // MN elements per atom
    static constexpr int GROUP = ES == 4 ? 4 : 8;                   // K rows per swizzle group
    static constexpr uint32_t SBO = GROUP * W;
    static constexpr uint32_t LAYOUT = ES == 4 ? 1u : (W == 64 ? 4u : 2u);
    static constexpr int TMA_SWIZZLE = ES == 4 ? int(CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)
                                               : (W == 64 ? int(CU_TENSOR_MAP_SWIZZLE_64B)
                                                          : int(CU_TENSOR_MAP_SWIZZLE_128B));
};

template <int ES, bool A_MN, bool B_MN, int BN>
__host__ __device__ constexpr uint32_t instr_desc() {
    // c_format F32 (bit 4), a/b format (bits 7-9 / 10-12): bf16 = 1, tf32 = 2,
    // a/b major (bits 15/16), N >> 3 (bits 17-22), M >> 4 (bits 24-28)
    return (1u << 4) | ((ES == 4 ? 2u : 1u) << 7) | ((ES == 4 ? 2u : 1u) << 10) |
           (uint32_t(A_MN) << 15) | (uint32_t(B_MN) << 16) | (uint32_t(BN >> 3) << 17) |
           (uint32_t(BM >> 4) << 24);
}

template <int ES>
__device__ __forceinline__ void mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                    uint32_t accumulate) {
    if constexpr (ES == 4) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
            :: "r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(accumulate) : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
            :: "r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(accumulate) : "memory");
    }
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// ------------------------------------------------------- TMA-store epilogue
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, uint32_t src, int c0, int c1,
                                             int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];"
                 :: "l"(reinterpret_cast<uint64_t>(map)), "r"(src), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory");
}
// Before the CTA exits: its bulk stores have finished reading shared memory
// (their global writes complete with the grid, as every kernel boundary and
// the split-K reduce's griddepcontrol.wait observe).
__device__ __forceinline__ void bulk_wait_smem_free() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// One epilogue warp stores its 32 rows x `cols` of the accumulator through
// TMA: per 32-column chunk, tcgen05.ld (lane = row), alpha, 8 STS.128 into a
// 128B-swizzled 32x32 buffer (chunk j of row r at r*128 + ((j ^ (r & 7)) << 4):
// the 8 lanes of a quarter-warp hit 8 distinct bank groups), then lane 0
// issues one bulk tensor store -- TMA clips rows / columns past the tensor,
// so no bounds checks -- double-buffered against the store still reading the
// other buffer.  `it` counts this warp's chunks across tiles.
__device__ __forceinline__ void tmem_ld32_async(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void epi_tma_tile(const CUtensorMap* map_c, uint32_t taddr, int cols,
                                             int n0, int row0, int bz, float alpha,
                                             uint32_t bufs, int lane, int& it,
                                             bool trace_warp = false) {
    // the next chunk's TMEM load is in flight while this one is staged
    uint32_t nxt[32];
    tmem_ld32_async(taddr, nxt);
#pragma unroll 1
    for (int c0 = 0; c0 < cols; c0 += 32, ++it) {
        tmem_wait_ld();
        // the registers are defined only after the wait: re-bind them here so
        // the compiler cannot read them before it
#pragma unroll
        for (int j = 0; j < 32; ++j) asm volatile("" : "+r"(nxt[j]));
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(nxt[j]);
        if (trace_warp && lane == 0 && c0 < 128) trace(8 + 2 * (c0 >> 5));
        if (c0 + 32 < cols) tmem_ld32_async(taddr + c0 + 32, nxt);
        const uint32_t buf = bufs + uint32_t(it & 1) * EPI_BUF;
        if (it >= 2) {  // the store issued from this buffer two chunks ago has read it
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
        }
        const uint32_t row = buf + uint32_t(lane) * 128u;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t addr = row + (uint32_t(j ^ (lane & 7)) << 4);
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};"
                         :: "r"(addr), "f"(alpha * v[4 * j]), "f"(alpha * v[4 * j + 1]),
                            "f"(alpha * v[4 * j + 2]), "f"(alpha * v[4 * j + 3]) : "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
            tma_store_3d(map_c, buf, n0 + c0, row0, bz);
            bulk_commit();
            if (trace_warp && c0 < 128) trace(9 + 2 * (c0 >> 5));
        }
    }
    tmem_wait_ld();  // (no load is outstanding here; keeps the fence before acc_empty honest)
}

// ------------------------------------------------------------------ kernel
// Tile t (0 <= t < tiles_m*tiles_n*batch): batch-major, then a grouped raster
// of GROUP_M m-tiles sweeping n inside each batch.
__device__ __forceinline__ void tile_coords(int t, const TcParams& p, int bn, int& m0, int& n0,
                                            int& bz) {
    const int per_batch = p.tiles_m * p.tiles_n;
    bz = t / per_batch;
    const int tile = t - bz * per_batch;
    const int per_group = p.group_m * p.tiles_n;
    const int group = tile / per_group;
    const int first_m = group * p.group_m;
    const int gsz = min(p.tiles_m - first_m, p.group_m);
    const int in_group = tile - group * per_group;
    m0 = (first_m + in_group % gsz) * BM;
    n0 = (in_group / gsz) * bn;
}

// NBUF = 1: one tile per CTA (grid = tiles). NBUF = 2: persistent CTAs (grid
// = SM count) striding over tiles with a double-buffered TMEM accumulator, so
// the epilogue of tile i overlaps the MMAs of tile i+1 and the TMA ring runs
// ahead across tile boundaries.
template <int ES, int BN, bool A_MN, bool B_MN, int NBUF>
__global__ void __launch_bounds__(NUM_THREADS, 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
               const __grid_constant__ CUtensorMap map_c, const TcParams p) {
    constexpr int ROW = 128;                  // bytes of K per operand row per stage
    constexpr int BK = ROW / ES;              // K elements per stage
    constexpr int UMMA_K = 32 / ES;           // K per tcgen05.mma
    using MA = MnMajor<ES, BM>;
    using MB = MnMajor<ES, BN>;
    constexpr uint32_t A_BYTES = BM * ROW;
    constexpr uint32_t B_BYTES = BN * ROW;
    constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
    constexpr uint32_t IDESC = instr_desc<ES, A_MN, B_MN, BN>();
    constexpr uint32_t TMEM_COLS = BN * NBUF;

    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte aligned stage ring, epilogue buffers (1024-aligned), barriers, TMEM slot
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + STAGE_ALIGN - 1) & ~uint32_t(STAGE_ALIGN - 1);
    uint8_t* gbase = smem_raw + (base - raw);
    const int S = p.stages;
    const uint32_t epi = base + S * STAGE_BYTES;
    float* staging = reinterpret_cast<float*>(gbase + S * STAGE_BYTES);
    // barriers: full[S], empty[S], acc_full[2], acc_empty[2]
    const uint32_t bars = epi + EPI_BYTES;
    uint32_t* tmem_slot =
        reinterpret_cast<uint32_t*>(gbase + S * STAGE_BYTES + EPI_BYTES + (2 * S + 4) * 8);
    auto full_bar = [&](int s) { return bars + 8u * s; };
    auto empty_bar = [&](int s) { return bars + 8u * (S + s); };
    auto acc_full = [&](int b) { return bars + 8u * (2 * S + b); };
    auto acc_empty = [&](int b) { return bars + 8u * (2 * S + 2 + b); };

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) trace(0);
    const int units = p.tiles_m * p.tiles_n * p.batch * p.splits;  // (tile, K split) work units
    // let the split-K reduce kernel's launch start now; its griddepcontrol.wait
    // still waits for this whole grid to finish and flush
    if (p.splits > 1) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(acc_full(b), 1);
            mbar_init(acc_empty(b), 4);  // one arrival per epilogue warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
        asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
        if (p.tma_store)
            asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(&map_c)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(smem_u32(tmem_slot)), "r"(TMEM_COLS) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) trace(1);

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer: one ring across all of this CTA's units
            int kt_all = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                int m0, n0, bz, kb0, kb1;
                tile_coords(u / p.splits, p, BN, m0, n0, bz);
                split_range(u % p.splits, p.splits, p.k_tiles, kb0, kb1);
                const int za = bz * p.a_batch, zb = bz * p.b_batch;
                for (int kt = kb0; kt < kb1; ++kt, ++kt_all) {
                    const int s = kt_all % S;
                    const uint32_t phase = (kt_all / S) & 1;
                    mbar_wait(empty_bar(s), phase ^ 1);
                    mbar_expect_tx(full_bar(s), STAGE_BYTES);
                    const uint32_t sa = base + s * STAGE_BYTES;
                    const uint32_t sb = sa + A_BYTES;
                    const int k0 = kt * BK;
                    if constexpr (!A_MN) {
                        tma_load_3d(sa, &map_a, k0, m0, za, full_bar(s));
                    } else {
#pragma unroll
                        for (int j = 0; j < BM / MA::ATOM; ++j)
                            tma_load_3d(sa + j * BK * MA::W, &map_a, m0 + j * MA::ATOM, k0, za,
                                        full_bar(s));
                    }
                    if constexpr (!B_MN) {
                        tma_load_3d(sb, &map_b, k0, n0, zb, full_bar(s));
                    } else {
#pragma unroll
                        for (int j = 0; j < BN / MB::ATOM; ++j)
                            tma_load_3d(sb + j * BK * MB::W, &map_b, n0 + j * MB::ATOM, k0, zb,
                                        full_bar(s));
                    }
                    if (kt_all == 0) trace(2);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            int kt_all = 0, it = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x, ++it) {
                int kb0, kb1;
                split_range(u % p.splits, p.splits, p.k_tiles, kb0, kb1);
                const int buf = NBUF == 2 ? (it & 1) : 0;
                const uint32_t use = NBUF == 2 ? ((it >> 1) & 1) : (it & 1);
                mbar_wait(acc_empty(buf), use ^ 1);  // epilogue drained this buffer
                fence_after_sync();
                const uint32_t d = tmem + uint32_t(buf * BN);
                for (int kt = kb0; kt < kb1; ++kt, ++kt_all) {
                    const int s = kt_all % S;
                    const uint32_t phase = (kt_all / S) & 1;
                    mbar_wait(full_bar(s), phase);
                    fence_after_sync();
                    if (kt_all == 0) trace(3);
                    const uint32_t sa = base + s * STAGE_BYTES;
                    const uint32_t sb = sa + A_BYTES;
#pragma unroll
                    for (int k = 0; k < BK / UMMA_K; ++k) {
                        // K-major: advance 32 B inside the 128B-swizzled row (8-row
                        // groups, SBO 1024); MN-major: advance UMMA_K rows of W bytes,
                        // LBO = one atom column block (BK rows), SBO = one swizzle group
                        const uint64_t da =
                            A_MN ? smem_desc(sa + k * UMMA_K * MA::W, BK * MA::W, MA::SBO, MA::LAYOUT)
                                 : smem_desc(sa + k * 32, 16, 1024, 2);
                        const uint64_t db =
                            B_MN ? smem_desc(sb + k * UMMA_K * MB::W, BK * MB::W, MB::SBO, MB::LAYOUT)
                                 : smem_desc(sb + k * 32, 16, 1024, 2);
                        mma<ES>(d, da, db, IDESC, (kt != kb0) || (k != 0));
                    }
                    umma_commit(empty_bar(s));  // frees the stage once these MMAs retire
                }
                umma_commit(acc_full(buf));     // accumulator of this tile complete
                trace(4);
            }
        }
    } else {  // ---- epilogue warps 2..5: TMEM lane quarter = warp % 4
        const int q = warp & 3;
        float* st = staging + (warp - 2) * 32 * EPI_PITCH;
        const uint32_t ebufs = epi + uint32_t(warp - 2) * 2 * EPI_BUF;
        int it = 0, eit = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++it) {
            const int t = u / p.splits;
            int m0, n0, bz;
            tile_coords(t, p, BN, m0, n0, bz);
            const int buf = NBUF == 2 ? (it & 1) : 0;
            const uint32_t use = NBUF == 2 ? ((it >> 1) & 1) : (it & 1);
            mbar_wait(acc_full(buf), use);
            fence_after_sync();
            if (warp == 2 && lane == 0) trace(5);
            float* Cb = p.C + int64_t(bz) * p.sc;
            const int row0 = m0 + q * 32;
            const uint32_t taddr = tmem + (uint32_t(q * 32) << 16) + uint32_t(buf * BN);
            const int cols = min(BN, p.N - n0);
            if (p.tma_store == 2) {  // split-K partial: ws tile (unit), rows q*32.., alpha later
                epi_tma_tile(&map_c, taddr, cols, 0, q * 32, t * p.splits + u % p.splits, 1.0f,
                             ebufs, lane, eit, warp == 2 && it == 0);
                if (warp == 2 && lane == 0) trace(6);
                fence_before_sync();
                if (lane == 0)
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(acc_empty(buf))
                                 : "memory");
                continue;
            }
            if (p.tma_store) {
                epi_tma_tile(&map_c, taddr, cols, n0, row0, bz, p.alpha, ebufs, lane, eit,
                             warp == 2 && it == 0);
                if (warp == 2 && lane == 0) trace(6);
                fence_before_sync();  // the tcgen05.ld of this tile are complete
                if (lane == 0)
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(acc_empty(buf))
                                 : "memory");
                continue;
            }
            // split-K: this unit's partial tile, full BM x BN, row-major
            float* part = p.splits > 1
                ? p.ws + (int64_t(t) * p.splits + u % p.splits) * (BM * BN) : nullptr;
#pragma unroll 1
            for (int c0 = 0; c0 < cols; c0 += 32) {
                float v[32];
                tmem_ld32(taddr + c0, v);
#pragma unroll
                for (int j = 0; j < 32; ++j) st[lane * EPI_PITCH + j] = v[j];
                __syncwarp();
                if (part) {
#pragma unroll 4
                    for (int r = 0; r < 32; ++r)
                        __stcg(part + (q * 32 + r) * BN + c0 + lane, st[r * EPI_PITCH + lane]);
                } else {
                    const int n = n0 + c0 + lane;
                    if (n < p.N) {
#pragma unroll 4
                        for (int r = 0; r < 32; ++r) {
                            const int m = row0 + r;
                            if (m < p.M) {
                                float* dst = Cb + int64_t(m) * p.ldc + n;
                                const float x = p.alpha * st[r * EPI_PITCH + lane];
                                *dst = p.beta == 0.0f ? x : fmaf(p.beta, *dst, x);
                            }
                        }
                    }
                }
                __syncwarp();
            }
            if (warp == 2 && lane == 0) trace(6);
            fence_before_sync();
            if (lane == 0) {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(acc_empty(buf))
                             : "memory");
            }
        }
    }
    if (p.tma_store && warp >= 2 && lane == 0) bulk_wait_smem_free();
    fence_before_sync();
    __syncthreads();
    if (warp == 1) {
        fence_after_sync();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem),
                     "r"(TMEM_COLS) : "memory");
    }
    if (threadIdx.x == 0) trace(7);
}

// Split-K reduction: one thread per 4 consecutive columns of one tile row;
// sums the S partials in split order, then alpha / beta and bounds.
template <int BN>
__global__ void __launch_bounds__(256)
tc_splitk_reduce(const TcParams p) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // partials complete and visible
    constexpr int C4 = BN / 4;                           // float4 columns per tile row
    const int64_t total = int64_t(p.tiles_m) * p.tiles_n * p.batch * BM * C4;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int c4 = int(i % C4);
        const int r = int((i / C4) % BM);
        const int t = int(i / (int64_t(C4) * BM));
        int m0, n0, bz;
        tile_coords(t, p, BN, m0, n0, bz);
        const int m = m0 + r, n = n0 + 4 * c4;
        if (m >= p.M || n >= p.N) continue;
        const float4* src = reinterpret_cast<const float4*>(
            p.ws + int64_t(t) * p.splits * (BM * BN) + r * BN) + c4;
        float4 acc = __ldcg(src);
        for (int sp = 1; sp < p.splits; ++sp) {
            const float4 v = __ldcg(src + int64_t(sp) * (BM * BN / 4));
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        float* dst = p.C + int64_t(bz) * p.sc + int64_t(m) * p.ldc + n;
        const float a4[4] = {acc.x, acc.y, acc.z, acc.w};
        const int cols = min(4, p.N - n);
        for (int j = 0; j < cols; ++j) {
            const float x = p.alpha * a4[j];
            dst[j] = p.beta == 0.0f ? x : fmaf(p.beta, dst[j], x);
        }
    }
}

// --------------------------------------------------------- 2-CTA kernel
// cta_group::2: a cluster of two CTAs (one TPC) computes a 256 x BN tile with
// M=256 tcgen05.mma issued by the even (leader) CTA. Each CTA stages its own
// 128 rows of A and half (BN/2) of B per stage -- the pair shares operands, so
// shared-memory fill traffic per MMA flop is 2/3 of the 1-CTA kernel's at
// BN = 256 -- and holds its 128 x BN half of D in its own TMEM. Both CTAs'
// TMA transactions complete on the leader's full barrier; the leader's
// tcgen05.commit multicasts to both CTAs' empty / acc_full barriers; both
// epilogues release the leader's acc_empty barrier. Persistent over tiles
// with a double-buffered accumulator, like the NBUF = 2 kernel.
__device__ __forceinline__ void tma_load_3d_pair(uint32_t dst, const CUtensorMap* map, int c0,
                                                 int c1, int c2, uint32_t leader_bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];"
        :: "r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2),
           "r"(leader_bar) : "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint32_t bar) {
    asm volatile(
        "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], m;\n\t}" :: "r"(bar) : "memory");
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
                 ::: "memory");
}
template <int ES>
__device__ __forceinline__ void mma_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
    if constexpr (ES == 4) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
            :: "r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(accumulate) : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
            :: "r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(accumulate) : "memory");
    }
}

constexpr uint32_t PEER_MASK = 0xFEFFFFFFu;  // shared::cluster address of the even CTA

template <int ES, int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
tc_gemm_pair_kernel(const __grid_constant__ CUtensorMap map_a,
                    const __grid_constant__ CUtensorMap map_b,
                    const __grid_constant__ CUtensorMap map_c, const TcParams p) {
    constexpr int ROW = 128;
    constexpr int BK = ROW / ES;
    constexpr int UMMA_K = 32 / ES;
    constexpr int HN = BN / 2;                   // B columns staged per CTA
    using MA = MnMajor<ES, BM>;
    using MB = MnMajor<ES, HN>;
    constexpr uint32_t A_BYTES = BM * ROW;
    constexpr uint32_t B_BYTES = HN * ROW;
    constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
    // M = 256 across the pair, N = BN
    constexpr uint32_t IDESC =
        (instr_desc<ES, A_MN, B_MN, BN>() & ~(0x1Fu << 24)) | (uint32_t(256 >> 4) << 24);
    constexpr uint32_t TMEM_COLS = 2 * BN;

    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + STAGE_ALIGN - 1) & ~uint32_t(STAGE_ALIGN - 1);
    uint8_t* gbase = smem_raw + (base - raw);
    const int S = p.stages;
    const uint32_t epi = base + S * STAGE_BYTES;
    float* staging = reinterpret_cast<float*>(gbase + S * STAGE_BYTES);
    const uint32_t bars = epi + EPI_BYTES;
    uint32_t* tmem_slot =
        reinterpret_cast<uint32_t*>(gbase + S * STAGE_BYTES + EPI_BYTES + (2 * S + 4) * 8);
    auto full_bar = [&](int s) { return bars + 8u * s; };
    auto empty_bar = [&](int s) { return bars + 8u * (S + s); };
    auto acc_full = [&](int b) { return bars + 8u * (2 * S + b); };
    auto acc_empty = [&](int b) { return bars + 8u * (2 * S + 2 + b); };

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    // pair tiles: 256-row m tiles (tiles_m counts them)
    const int total = p.tiles_m * p.tiles_n * p.batch;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(acc_full(b), 1);
            mbar_init(acc_empty(b), 8);  // 4 epilogue warps x 2 CTAs
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
        asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
        if (p.tma_store)
            asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(&map_c)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(smem_u32(tmem_slot)), "r"(TMEM_COLS) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    fence_before_sync();
    cluster_sync();  // both CTAs' barriers exist before any remote arrive / multicast
    fence_after_sync();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer (both CTAs; bytes land on the leader's barrier)
            int kt_all = 0;
            for (int t = pair; t < total; t += npairs) {
                int m0, n0, bz;
                tile_coords(t, p, BN, m0, n0, bz);  // m0 in units of BM*2 below
                m0 = m0 * 2 + int(rank) * BM;
                const int nb = n0 + int(rank) * HN;
                const int za = bz * p.a_batch, zb = bz * p.b_batch;
                for (int kt = 0; kt < p.k_tiles; ++kt, ++kt_all) {
                    const int s = kt_all % S;
                    const uint32_t phase = (kt_all / S) & 1;
                    mbar_wait(empty_bar(s), phase ^ 1);
                    const uint32_t lbar = full_bar(s) & PEER_MASK;
                    if (leader) mbar_expect_tx(full_bar(s), 2 * STAGE_BYTES);
                    const uint32_t sa = base + s * STAGE_BYTES;
                    const uint32_t sb = sa + A_BYTES;
                    const int k0 = kt * BK;
                    if constexpr (!A_MN) {
                        tma_load_3d_pair(sa, &map_a, k0, m0, za, lbar);
                    } else {
#pragma unroll
                        for (int j = 0; j < BM / MA::ATOM; ++j)
                            tma_load_3d_pair(sa + j * BK * MA::W, &map_a, m0 + j * MA::ATOM, k0, za,
                                             lbar);
                    }
                    if constexpr (!B_MN) {
                        tma_load_3d_pair(sb, &map_b, k0, nb, zb, lbar);
                    } else {
#pragma unroll
                        for (int j = 0; j < HN / MB::ATOM; ++j)
                            tma_load_3d_pair(sb + j * BK * MB::W, &map_b, nb + j * MB::ATOM, k0, zb,
                                             lbar);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && leader) {  // ---- MMA issuer (leader only)
            int kt_all = 0, it = 0;
            for (int t = pair; t < total; t += npairs, ++it) {
                const int buf = it & 1;
                const uint32_t use = (it >> 1) & 1;
                mbar_wait(acc_empty(buf), use ^ 1);
                fence_after_sync();
                const uint32_t d = tmem + uint32_t(buf * BN);
                for (int kt = 0; kt < p.k_tiles; ++kt, ++kt_all) {
                    const int s = kt_all % S;
                    const uint32_t phase = (kt_all / S) & 1;
                    mbar_wait(full_bar(s), phase);
                    fence_after_sync();
                    const uint32_t sa = base + s * STAGE_BYTES;
                    const uint32_t sb = sa + A_BYTES;
#pragma unroll
                    for (int k = 0; k < BK / UMMA_K; ++k) {
                        const uint64_t da =
                            A_MN ? smem_desc(sa + k * UMMA_K * MA::W, BK * MA::W, MA::SBO, MA::LAYOUT)
                                 : smem_desc(sa + k * 32, 16, 1024, 2);
                        const uint64_t db =
                            B_MN ? smem_desc(sb + k * UMMA_K * MB::W, BK * MB::W, MB::SBO, MB::LAYOUT)
                                 : smem_desc(sb + k * 32, 16, 1024, 2);
                        mma_pair<ES>(d, da, db, IDESC, (kt | k) != 0);
                    }
                    umma_commit_pair(empty_bar(s));   // frees stage s in both CTAs
                }
                umma_commit_pair(acc_full(buf));      // both halves of D complete
            }
        }
    } else {  // ---- epilogue warps 2..5 of both CTAs: own 128 rows of D
        const int q = warp & 3;
        float* st = staging + (warp - 2) * 32 * EPI_PITCH;
        const uint32_t ebufs = epi + uint32_t(warp - 2) * 2 * EPI_BUF;
        int it = 0, eit = 0;
        for (int t = pair; t < total; t += npairs, ++it) {
            int m0, n0, bz;
            tile_coords(t, p, BN, m0, n0, bz);
            m0 = m0 * 2 + int(rank) * BM;
            const int buf = it & 1;
            const uint32_t use = (it >> 1) & 1;
            mbar_wait(acc_full(buf), use);
            fence_after_sync();
            float* Cb = p.C + int64_t(bz) * p.sc;
            const int row0 = m0 + q * 32;
            const uint32_t taddr = tmem + (uint32_t(q * 32) << 16) + uint32_t(buf * BN);
            const int cols = min(BN, p.N - n0);
            if (p.tma_store) {
                epi_tma_tile(&map_c, taddr, cols, n0, row0, bz, p.alpha, ebufs, lane, eit);
                fence_before_sync();
                if (lane == 0)
                    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];"
                                 :: "r"(acc_empty(buf) & PEER_MASK) : "memory");
                continue;
            }
#pragma unroll 1
            for (int c0 = 0; c0 < cols; c0 += 32) {
                float v[32];
                tmem_ld32(taddr + c0, v);
#pragma unroll
                for (int j = 0; j < 32; ++j) st[lane * EPI_PITCH + j] = v[j];
                __syncwarp();
                const int n = n0 + c0 + lane;
                if (n < p.N) {
#pragma unroll 4
                    for (int r = 0; r < 32; ++r) {
                        const int m = row0 + r;
                        if (m < p.M) {
                            float* dst = Cb + int64_t(m) * p.ldc + n;
                            const float x = p.alpha * st[r * EPI_PITCH + lane];
                            *dst = p.beta == 0.0f ? x : fmaf(p.beta, *dst, x);
                        }
                    }
                }
                __syncwarp();
            }
            fence_before_sync();
            if (lane == 0) {
                asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];"
                             :: "r"(acc_empty(buf) & PEER_MASK) : "memory");
            }
        }
    }
    if (p.tma_store && warp >= 2 && lane == 0) bulk_wait_smem_free();
    fence_before_sync();
    __syncthreads();
    cluster_sync();
    if (warp == 1) {
        fence_after_sync();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tmem),
                     "r"(TMEM_COLS) : "memory");
    }
}

// ------------------------------------------------------------------- host
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encoder() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess && q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(ptr);
    });
    return fn;
}

// 3-D tensor map over (inner, outer, batch) with a 128-byte swizzled box.
// Encoded maps are cached per host thread (a small direct-mapped table keyed
// by every encode argument): cuTensorMapEncodeTiled costs microseconds, and a
// GEMM launch needs up to three of them -- on small problems the host enqueue,
// not the kernel, would otherwise set the launch rate.  A map depends only on
// its arguments (address, extents, strides, box, swizzle), so a hit is exact.
struct MapKey {
    const void* ptr;
    int64_t inner, outer, batch, ld, bstride;
    int box_inner, box_outer, swizzle, bf16;
    bool operator==(const MapKey& o) const { return std::memcmp(this, &o, sizeof *this) == 0; }
};
struct MapSlot {
    MapKey key;
    CUtensorMap map;
    bool valid;
};

static kp_status make_map(CUtensorMap* map, bool bf16, const void* ptr, int64_t inner,
                          int64_t outer, int64_t batch, int64_t ld, int64_t bstride, int box_inner,
                          int box_outer, int swizzle) {
    MapKey key;
    std::memset(&key, 0, sizeof key);  // padding bytes take part in the comparison
    key.ptr = ptr; key.inner = inner; key.outer = outer; key.batch = batch; key.ld = ld;
    key.bstride = batch > 1 ? bstride : 0; key.box_inner = box_inner; key.box_outer = box_outer;
    key.swizzle = swizzle; key.bf16 = bf16;
    constexpr int SLOTS = 64;
    static thread_local MapSlot cache[SLOTS];
    uint64_t h = reinterpret_cast<uintptr_t>(ptr) >> 4;
    h = h * 0x9E3779B97F4A7C15ull ^ uint64_t(inner) * 31 ^ uint64_t(outer) * 131 ^
        uint64_t(box_inner) * 7 ^ uint64_t(box_outer) * 13 ^ uint64_t(ld) * 17 ^ uint64_t(swizzle);
    MapSlot& slot = cache[(h ^ (h >> 29)) % SLOTS];
    if (slot.valid && slot.key == key) {
        *map = slot.map;
        return KP_OK;
    }
    EncodeFn enc = encoder();
    if (!enc) return fail(KP_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
    const int es = bf16 ? 2 : 4;
    cuuint64_t dims[3] = {cuuint64_t(inner), cuuint64_t(outer), cuuint64_t(batch)};
    cuuint64_t strides[2] = {cuuint64_t(ld * es), cuuint64_t((batch > 1 ? bstride : outer * ld) * es)};
    cuuint32_t box[3] = {cuuint32_t(box_inner), cuuint32_t(box_outer), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = enc(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                           3, const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CUtensorMapSwizzle(swizzle),
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(KP_ERR_ALIGNMENT, "cuTensorMapEncodeTiled rejected the operand");
    slot.key = key;
    slot.map = *map;
    slot.valid = true;
    return KP_OK;
}

static const uint32_t kTiles[4] = {1, 2, 4, 8};
static int tidx(uint32_t v) {
    for (int i = 0; i < 4; ++i)
        if (kTiles[i] == v) return i;
    return -1;
}

// Config list per family (canonical KernelConfig order):
//   (acc, 1, ct, 8, 8)    one 128 x BN tile per CTA
//   (acc, 1, ct, 16, 16)  persistent CTAs, double-buffered TMEM accumulator
//   (acc, 2, ct, 16, 16)  persistent CTA pairs (cta_group::2, M = 256), ct in {4, 8}
static int tc_config_table(kp_config* out) {
    int n = 0;
    for (int a = 0; a < 4; ++a) {
        for (int c = 0; c < 4; ++c) {
            out[n++] = kp_config{kTiles[a], 1u, kTiles[c], 8u, 8u};
            out[n++] = kp_config{kTiles[a], 1u, kTiles[c], 16u, 16u};
        }
        for (int c = 2; c < 4; ++c) out[n++] = kp_config{kTiles[a], 2u, kTiles[c], 16u, 16u};
    }
    return n;
}

int32_t num_configs(kp_family fam) { return (fam == KP_TF32_TC || fam == KP_BF16_TC) ? 40 : 0; }

kp_status config_at(kp_family fam, int32_t index, kp_config* out) {
    if (index < 0 || index >= num_configs(fam)) return fail(KP_ERR_INVALID_ARG, "config index out of range");
    kp_config table[40];
    tc_config_table(table);
    *out = table[index];
    return KP_OK;
}

kp_status valid(kp_family fam, const kp_config& c) {
    if (num_configs(fam) == 0) return fail(KP_ERR_INVALID_ARG, "not a tensor-core family");
    kp_config table[40];
    const int n = tc_config_table(table);
    for (int i = 0; i < n; ++i)
        if (std::memcmp(&table[i], &c, sizeof c) == 0) return KP_OK;
    return fail(KP_ERR_INVALID_CONFIG,
                "tcgen05 family configs: (acc, 1, ct, 8, 8), (acc, 1, ct, 16, 16), "
                "(acc, 2, ct in 4|8, 16, 16); acc, ct in 1,2,4,8");
}

static size_t smem_bytes(int bn, int stages) {
    return STAGE_ALIGN + size_t(stages) * (BM + bn) * 128 + EPI_BYTES + (2 * stages + 6) * 8;
}

static int sm_count() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// Raster group height (m-tiles sharing one sweep over n).  KP_TC_GROUP_M
// overrides it for tuning experiments only (never set by the library).
static int group_m() {
    static const int g = [] {
        const char* e = std::getenv("KP_TC_GROUP_M");
        const int v = e ? std::atoi(e) : 0;
        return v > 0 ? v : GROUP_M;
    }();
    return g;
}

// ---------------------------------------------------------- split-K state
// Per-device workspace: WS_SLOTS slots of WS_SLOT_BYTES of partial tiles.
// Launches take slots round-robin, so up to WS_SLOTS split-K GEMMs in flight
// on different streams never share a slot.
constexpr int WS_SLOTS = 4;
constexpr size_t WS_SLOT_BYTES = size_t(64) << 20;
static std::atomic<int> g_split_mode{1};

int32_t set_split_mode(int32_t mode) {
    if (mode < 0 || mode > 64) return -1;
    return g_split_mode.exchange(mode);
}

static kp_status ws_reserve(float** ws) {
    static std::mutex mu;
    static char* base[64] = {nullptr};
    static unsigned next[64] = {0};
    const int dev = current_device();
    if (dev < 0 || dev >= 64) return fail(KP_ERR_CUDA, "split-K: bad device");
    std::lock_guard<std::mutex> lock(mu);
    if (!base[dev]) {
        void* ptr = nullptr;
        if (cudaMalloc(&ptr, WS_SLOTS * WS_SLOT_BYTES) != cudaSuccess)
            return check_launch("split-K workspace cudaMalloc");
        base[dev] = static_cast<char*>(ptr);
    }
    *ws = reinterpret_cast<float*>(base[dev] + (next[dev]++ % WS_SLOTS) * WS_SLOT_BYTES);
    return KP_OK;
}

// K splits for a grid of `tiles` 128 x bn tiles over k_tiles K stages.
// Auto (mode 1): only grids filling under half the SMs split, into as many
// ranges as one wave of units allows while every range keeps >= 4 k-tiles
// (the TMA ring's fill must stay amortised); mode >= 2 forces that many
// splits (tests); mode 0 never splits.
static int choose_splits(int64_t tiles, int k_tiles, int bn) {
    const int mode = g_split_mode.load(std::memory_order_relaxed);
    if (mode == 0) return 1;
    int64_t S;
    if (mode >= 2) {
        S = mode;
    } else {
        const int sms = sm_count();
        if (tiles * 2 > sms) return 1;
        S = std::min<int64_t>(sms / tiles, k_tiles / 4);
    }
    S = std::min<int64_t>(S, k_tiles);
    S = std::min<int64_t>(S, int64_t(WS_SLOT_BYTES / (size_t(BM) * bn * sizeof(float))) / tiles);
    return S < 2 ? 1 : int(S);
}

// TMA-store epilogue eligibility + C tensor map (fp32, 32x32 boxes, 128B
// swizzle): beta == 0 (C write-only), 16-byte aligned C rows / batches, and
// no split-K (partials take the workspace path).  KP_TC_TMA_STORE=0 turns it
// off for A/B timing (tuning experiments only).
static bool tma_store_on() {
    static const bool on = [] {
        const char* e = std::getenv("KP_TC_TMA_STORE");
        return !(e && e[0] == '0');
    }();
    return on;
}
static kp_status c_map(const GemmProblem& g, int splits, CUtensorMap* mc, int* use) {
    std::memset(mc, 0, sizeof *mc);
    *use = 0;
    if (splits > 1) return KP_OK;  // see ws_map
    if (!tma_store_on() || g.beta != 0.0f || !aligned16(g.C) || (g.ldc * 4) % 16 ||
        (g.batch > 1 && (g.sc * 4) % 16))
        return KP_OK;
    kp_status st = make_map(mc, false, g.C, g.n, g.m, g.batch, g.ldc, g.sc, 32, 32,
                            int(CU_TENSOR_MAP_SWIZZLE_128B));
    if (st != KP_OK) return st;
    *use = 1;
    return KP_OK;
}

// Split-K partial tiles [unit][BM][BN] of the workspace as a 3-D fp32 tensor
// (32x32 boxes, 128B swizzle) for the TMA-store epilogue.
static kp_status ws_map(float* ws, int bn, int64_t units, CUtensorMap* mc, int* use) {
    std::memset(mc, 0, sizeof *mc);
    *use = 0;
    if (!tma_store_on()) return KP_OK;
    kp_status st = make_map(mc, false, ws, bn, BM, units, bn, int64_t(BM) * bn, 32, 32,
                            int(CU_TENSOR_MAP_SWIZZLE_128B));
    if (st != KP_OK) return st;
    *use = 2;
    return KP_OK;
}

template <int ES, int BN, bool A_MN, bool B_MN, int NBUF>
static kp_status launch_t(const GemmProblem& g, int want_stages, cudaStream_t stream) {
    int stages = want_stages;
    while (stages > 2 && smem_bytes(BN, stages) > 227 * 1024) --stages;
    const size_t smem = smem_bytes(BN, stages);
    const bool bf16 = ES == 2;
    const int BK = 128 / ES;
    CUtensorMap ma, mb;
    kp_status st;
    const int64_t bat_a = g.sa ? g.batch : 1, bat_b = g.sb ? g.batch : 1;
    using MA = MnMajor<ES, BM>;
    using MB = MnMajor<ES, BN>;
    const int sw128 = int(CU_TENSOR_MAP_SWIZZLE_128B);
    if (!A_MN) st = make_map(&ma, bf16, g.A, g.k, g.m, bat_a, g.lda, g.sa, BK, BM, sw128);
    else       st = make_map(&ma, bf16, g.A, g.m, g.k, bat_a, g.lda, g.sa, MA::ATOM, BK, MA::TMA_SWIZZLE);
    if (st != KP_OK) return st;
    if (!B_MN) st = make_map(&mb, bf16, g.B, g.k, g.n, bat_b, g.ldb, g.sb, BK, BN, sw128);
    else       st = make_map(&mb, bf16, g.B, g.n, g.k, bat_b, g.ldb, g.sb, MB::ATOM, BK, MB::TMA_SWIZZLE);
    if (st != KP_OK) return st;
    auto kern = tc_gemm_kernel<ES, BN, A_MN, B_MN, NBUF>;
    static std::atomic<uint64_t> attr_set{0};  // per-device opt-in to > 48 KB dynamic smem
    const uint64_t dev_bit = uint64_t(1) << (current_device() & 63);
    if (!(attr_set.load(std::memory_order_acquire) & dev_bit)) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess)
            return check_launch("cudaFuncSetAttribute");
        attr_set.fetch_or(dev_bit, std::memory_order_release);
    }
    TcParams p;
    p.C = g.C;
    p.M = int(g.m); p.N = int(g.n); p.K = int(g.k);
    p.ldc = g.ldc; p.sc = g.sc;
    p.alpha = g.alpha; p.beta = g.beta;
    p.tiles_m = int((g.m + BM - 1) / BM);
    p.tiles_n = int((g.n + BN - 1) / BN);
    p.stages = stages;
    p.k_tiles = int((g.k + BK - 1) / BK);
    p.batch = int(g.batch);
    p.a_batch = g.sa ? 1 : 0;
    p.b_batch = g.sb ? 1 : 0;
    const int64_t tiles = int64_t(p.tiles_m) * p.tiles_n * g.batch;
    if (tiles > 0x7fffffffLL) return fail(KP_ERR_BAD_SHAPE, "tc: grid too large");
    p.splits = choose_splits(tiles, p.k_tiles, BN);
    p.group_m = group_m();
    p.ws = nullptr;
    if (p.splits > 1 && (st = ws_reserve(&p.ws)) != KP_OK) return st;
    CUtensorMap mc;
    const int64_t units = tiles * p.splits;
    if (p.splits > 1) st = ws_map(p.ws, BN, units, &mc, &p.tma_store);
    else st = c_map(g, p.splits, &mc, &p.tma_store);
    if (st != KP_OK) return st;
    const int64_t grid = NBUF == 2 ? std::min<int64_t>(units, sm_count()) : units;
    kern<<<dim3(unsigned(grid)), NUM_THREADS, smem, stream>>>(ma, mb, mc, p);
    note_launch();
    if ((st = check_launch("tc_gemm_kernel")) != KP_OK || p.splits == 1) return st;
    // split-K: reduce the partials (programmatic dependent launch)
    const int64_t work = tiles * BM * (BN / 4);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(std::min<int64_t>((work + 255) / 256, int64_t(sm_count()) * 8)));
    cfg.blockDim = dim3(256);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, tc_splitk_reduce<BN>, p) != cudaSuccess)
        return check_launch("tc_splitk_reduce");
    note_launch();
    return check_launch("tc_splitk_reduce");
}

static size_t pair_smem_bytes(int bn, int stages) {
    return STAGE_ALIGN + size_t(stages) * (BM + bn / 2) * 128 + EPI_BYTES + (2 * stages + 6) * 8;
}

template <int ES, int BN, bool A_MN, bool B_MN>
static kp_status launch_pair(const GemmProblem& g, int want_stages, cudaStream_t stream) {
    int stages = want_stages;
    while (stages > 2 && pair_smem_bytes(BN, stages) > 227 * 1024) --stages;
    const size_t smem = pair_smem_bytes(BN, stages);
    const bool bf16 = ES == 2;
    const int BK = 128 / ES;
    constexpr int HN = BN / 2;
    CUtensorMap ma, mb;
    kp_status st;
    const int64_t bat_a = g.sa ? g.batch : 1, bat_b = g.sb ? g.batch : 1;
    using MA = MnMajor<ES, BM>;
    using MB = MnMajor<ES, HN>;
    const int sw128 = int(CU_TENSOR_MAP_SWIZZLE_128B);
    if (!A_MN) st = make_map(&ma, bf16, g.A, g.k, g.m, bat_a, g.lda, g.sa, BK, BM, sw128);
    else       st = make_map(&ma, bf16, g.A, g.m, g.k, bat_a, g.lda, g.sa, MA::ATOM, BK, MA::TMA_SWIZZLE);
    if (st != KP_OK) return st;
    if (!B_MN) st = make_map(&mb, bf16, g.B, g.k, g.n, bat_b, g.ldb, g.sb, BK, HN, sw128);
    else       st = make_map(&mb, bf16, g.B, g.n, g.k, bat_b, g.ldb, g.sb, MB::ATOM, BK, MB::TMA_SWIZZLE);
    if (st != KP_OK) return st;
    auto kern = tc_gemm_pair_kernel<ES, BN, A_MN, B_MN>;
    static std::atomic<uint64_t> attr_set{0};  // per-device opt-in to > 48 KB dynamic smem
    const uint64_t dev_bit = uint64_t(1) << (current_device() & 63);
    if (!(attr_set.load(std::memory_order_acquire) & dev_bit)) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess)
            return check_launch("cudaFuncSetAttribute");
        attr_set.fetch_or(dev_bit, std::memory_order_release);
    }
    TcParams p;
    p.C = g.C;
    p.M = int(g.m); p.N = int(g.n); p.K = int(g.k);
    p.ldc = g.ldc; p.sc = g.sc;
    p.alpha = g.alpha; p.beta = g.beta;
    p.splits = 1;  // the pair kernel never splits K
    p.group_m = group_m();
    p.ws = nullptr;
    p.tiles_m = int((g.m + 2 * BM - 1) / (2 * BM));  // 256-row pair tiles
    p.tiles_n = int((g.n + BN - 1) / BN);
    p.stages = stages;
    p.k_tiles = int((g.k + BK - 1) / BK);
    p.batch = int(g.batch);
    p.a_batch = g.sa ? 1 : 0;
    p.b_batch = g.sb ? 1 : 0;
    const int64_t tiles = int64_t(p.tiles_m) * p.tiles_n * g.batch;
    if (tiles > 0x3fffffffLL) return fail(KP_ERR_BAD_SHAPE, "tc: grid too large");
    const int64_t pairs = std::min<int64_t>(tiles, sm_count() / 2);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(2 * pairs));
    cfg.blockDim = dim3(NUM_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CUtensorMap mc;
    if ((st = c_map(g, 1, &mc, &p.tma_store)) != KP_OK) return st;
    if (cudaLaunchKernelEx(&cfg, kern, ma, mb, mc, p) != cudaSuccess) return check_launch("tc_gemm_pair_kernel");
    note_launch();
    return check_launch("tc_gemm_pair_kernel");
}

// Lean library (the paper's deployment build, KP_LEAN): only the kernel
// instantiations the compiled selectors can return exist; the generated
// generated/tc_lean.h lists them as (es, bn, a_mn, b_mn, kind) with kind
// 1 = one tile per CTA, 2 = persistent, 3 = CTA pair.
#ifdef KP_LEAN
#include "generated/tc_lean.h"
#else
constexpr bool lean_allowed(int, int, bool, bool, int) { return true; }
#endif

template <int ES, int BN, bool A_MN, bool B_MN>
static kp_status pair_checked(const GemmProblem& g, int stages, cudaStream_t s) {
    if constexpr (lean_allowed(ES, BN, A_MN, B_MN, 3))
        return launch_pair<ES, BN, A_MN, B_MN>(g, stages, s);
    else
        return fail(KP_ERR_UNSUPPORTED, "kernel not in the lean library");
}

template <int ES, int BN, bool A_MN, bool B_MN, int NBUF>
static kp_status tile_checked(const GemmProblem& g, int stages, cudaStream_t s) {
    if constexpr (lean_allowed(ES, BN, A_MN, B_MN, NBUF))
        return launch_t<ES, BN, A_MN, B_MN, NBUF>(g, stages, s);
    else
        return fail(KP_ERR_UNSUPPORTED, "kernel not in the lean library");
}

template <int ES, int BN>
static kp_status by_layout_pair(const GemmProblem& g, int stages, cudaStream_t s) {
    if (!g.ta && g.tb) return pair_checked<ES, BN, false, false>(g, stages, s);
    if (!g.ta && !g.tb) return pair_checked<ES, BN, false, true>(g, stages, s);
    if (g.ta && g.tb) return pair_checked<ES, BN, true, false>(g, stages, s);
    return pair_checked<ES, BN, true, true>(g, stages, s);
}

template <int ES>
static kp_status by_tile_pair(const kp_config& c, const GemmProblem& g, cudaStream_t s) {
    static const int kStages[4] = {2, 3, 4, 6};
    const int stages = kStages[tidx(c.acc)];
    if (c.col_tile == 4) return by_layout_pair<ES, 128>(g, stages, s);
    return by_layout_pair<ES, 256>(g, stages, s);
}

template <int ES, int BN, int NBUF>
static kp_status by_layout(const GemmProblem& g, int stages, cudaStream_t s) {
    // A normal = K-major, A transposed = MN-major; B transposed = K-major, B normal = MN-major
    if (!g.ta && g.tb) return tile_checked<ES, BN, false, false, NBUF>(g, stages, s);
    if (!g.ta && !g.tb) return tile_checked<ES, BN, false, true, NBUF>(g, stages, s);
    if (g.ta && g.tb) return tile_checked<ES, BN, true, false, NBUF>(g, stages, s);
    return tile_checked<ES, BN, true, true, NBUF>(g, stages, s);
}

template <int ES, int NBUF>
static kp_status by_tile(const kp_config& c, const GemmProblem& g, cudaStream_t s) {
    static const int kStages[4] = {2, 3, 4, 6};
    const int stages = kStages[tidx(c.acc)];
    switch (c.col_tile) {
        case 1: return by_layout<ES, 32, NBUF>(g, stages, s);
        case 2: return by_layout<ES, 64, NBUF>(g, stages, s);
        case 4: return by_layout<ES, 128, NBUF>(g, stages, s);
        case 8: return by_layout<ES, 256, NBUF>(g, stages, s);
    }
    return fail(KP_ERR_INVALID_CONFIG, "tc: bad col_tile");
}

// ------------------------------------------------ unaligned-operand staging
// TMA needs 16-byte aligned bases and row / batch pitches.  An operand that
// has neither (K = 27 im2col rows, odd leading dimensions, offset views) is
// copied into a stream-ordered temporary (cudaMallocAsync from the device's
// default pool, freed with cudaFreeAsync after the GEMM) whose rows are padded
// to 16 bytes with zeros; the GEMM then runs on the copy with the same
// logical shape, so only the staging bytes are extra.
template <typename T>
__global__ void __launch_bounds__(256)
stage_rows_kernel(const T* __restrict__ src, T* __restrict__ dst, int64_t rows, int64_t cols,
                  int64_t ld, int64_t bstride, int64_t ld_dst, int64_t batch) {
    const int64_t per = rows * ld_dst, total = per * batch;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t b = i / per, e = i - b * per;
        const int64_t r = e / ld_dst, c = e - r * ld_dst;
        dst[i] = c < cols ? src[b * bstride + r * ld + c] : T(0.0f);
    }
}

static kp_status stage_operand(bool bf16, const void* src, int64_t rows, int64_t cols, int64_t ld,
                               int64_t bstride, int64_t batch, cudaStream_t s, void** out,
                               int64_t* ld_out, int64_t* bstride_out) {
    const int es = bf16 ? 2 : 4;
    const int64_t ld2 = (cols + 16 / es - 1) / (16 / es) * (16 / es);
    const int64_t bat = bstride ? batch : 1;  // a broadcast operand is staged once
    const size_t bytes = size_t(bat) * rows * ld2 * es;
    static std::once_flag pool_once[64];
    const int dev = current_device();
    std::call_once(pool_once[dev & 63], [dev] {  // keep freed staging memory pooled
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = ~uint64_t(0);
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    });
    if (cudaMallocAsync(out, bytes, s) != cudaSuccess) return check_launch("tc staging cudaMallocAsync");
    const int64_t total = int64_t(bat) * rows * ld2;
    const unsigned grid = unsigned(std::min<int64_t>((total + 255) / 256, int64_t(sm_count()) * 16));
    if (bf16)
        stage_rows_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(
            static_cast<const __nv_bfloat16*>(src), static_cast<__nv_bfloat16*>(*out), rows, cols,
            ld, bstride, ld2, bat);
    else
        stage_rows_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(src),
                                                      static_cast<float*>(*out), rows, cols, ld,
                                                      bstride, ld2, bat);
    note_launch();
    *ld_out = ld2;
    *bstride_out = bstride ? rows * ld2 : 0;
    return check_launch("stage_rows_kernel");
}

// TF32 with both operands MN-major (A transposed, B normal: the TN layout)
// runs the tensor pipe at ~52 % where any layout with a K-major operand runs
// at ~66 % (ncu, 4096^3; BF16 TN is unaffected): the 32-byte-granular
// MN-major swizzle on both sides.  Large TN problems therefore get A copied
// K-major first (tiled transpose into a stream-ordered temporary, 16-byte
// row pitch), which costs 2*m*k*4 bytes of traffic against the MMA time it
// saves; small ones keep the direct path.
__global__ void __launch_bounds__(256)
transpose_f32_kernel(const float* __restrict__ src, float* __restrict__ dst, int64_t rows,
                     int64_t cols, int64_t lds, int64_t ldd) {
    // src: rows x cols (row pitch lds); dst: cols x rows (row pitch ldd)
    __shared__ float tile[32][33];
    const int64_t r0 = int64_t(blockIdx.y) * 32, c0 = int64_t(blockIdx.x) * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
#pragma unroll
    for (int i = 0; i < 32; i += 8) {
        const int64_t r = r0 + ty + i, c = c0 + tx;
        tile[ty + i][tx] = (r < rows && c < cols) ? src[r * lds + c] : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 32; i += 8) {
        const int64_t c = c0 + ty + i, r = r0 + tx;
        if (c < cols && r < rows) dst[c * ldd + r] = tile[tx][ty + i];
    }
}

static bool tf32_tn_transpose(kp_family fam, const GemmProblem& g) {
    static const bool on = [] {
        const char* e = std::getenv("KP_TC_TN_TRANSPOSE");
        return !(e && e[0] == '0');
    }();
    // measured: 4096^3 291 -> 266 us, 8192^3 1862 -> 1695 us (= the NN
    // layout's time plus the copy); 2048^3 45 -> 50 us, so large problems only
    return on && fam == KP_TF32_TC && g.ta && !g.tb && g.batch == 1 && g.m >= 4096 &&
           g.n >= 4096 && g.k >= 2048;
}

kp_status launch(kp_family fam, const kp_config& c, const GemmProblem& g, cudaStream_t s) {
    kp_status st = valid(fam, c);
    if (st != KP_OK) return st;
    if (tf32_tn_transpose(fam, g)) {
        GemmProblem h = g;
        h.ta = false;
        h.lda = (g.k + 3) / 4 * 4;  // A' = op(A) stored m x k, K-major
        h.sa = 0;
        void* tmp = nullptr;
        if (cudaMallocAsync(&tmp, size_t(g.m) * h.lda * 4, s) != cudaSuccess)
            return check_launch("tc transpose cudaMallocAsync");
        // A stored k x m (row pitch lda) -> A' m x k
        const dim3 grid(unsigned((g.m + 31) / 32), unsigned((g.k + 31) / 32));
        transpose_f32_kernel<<<grid, 256, 0, s>>>(static_cast<const float*>(g.A),
                                                   static_cast<float*>(tmp), g.k, g.m, g.lda,
                                                   h.lda);
        note_launch();
        st = check_launch("transpose_f32_kernel");
        h.A = tmp;
        if (st == KP_OK) st = launch(fam, c, h, s);
        cudaFreeAsync(tmp, s);
        return st;
    }
    const int es = fam == KP_BF16_TC ? 2 : 4;
    auto al = [&](const void* ptr, int64_t ld, int64_t bs) {
        return aligned16(ptr) && (ld * es) % 16 == 0 && (g.batch == 1 || (bs * es) % 16 == 0);
    };
    const bool a_ok = al(g.A, g.lda, g.sa), b_ok = al(g.B, g.ldb, g.sb);
    if (!a_ok || !b_ok) {
        GemmProblem h = g;
        void* tmp[2] = {nullptr, nullptr};
        const bool bf16 = fam == KP_BF16_TC;
        if (!a_ok)
            st = stage_operand(bf16, g.A, g.ta ? g.k : g.m, g.ta ? g.m : g.k, g.lda, g.sa, g.batch,
                               s, &tmp[0], &h.lda, &h.sa);
        if (st == KP_OK && !b_ok)
            st = stage_operand(bf16, g.B, g.tb ? g.n : g.k, g.tb ? g.k : g.n, g.ldb, g.sb, g.batch,
                               s, &tmp[1], &h.ldb, &h.sb);
        if (tmp[0]) h.A = tmp[0];
        if (tmp[1]) h.B = tmp[1];
        if (st == KP_OK) st = launch(fam, c, h, s);
        for (void* t : tmp)
            if (t) cudaFreeAsync(t, s);
        return st;
    }
    if (c.row_tile == 2) return fam == KP_BF16_TC ? by_tile_pair<2>(c, g, s) : by_tile_pair<4>(c, g, s);
    const bool persistent = c.wg_rows == 16;
    if (fam == KP_BF16_TC) return persistent ? by_tile<2, 2>(c, g, s) : by_tile<2, 1>(c, g, s);
    return persistent ? by_tile<4, 2>(c, g, s) : by_tile<4, 1>(c, g, s);
}

}  // namespace tc
}  // namespace kp

#ifdef KP_TC_DEBUG
// Phase timestamps of the last traced launch (KP_TC_DEBUG builds only; not
// part of include/kp_abi.h): rows of 8 ns timestamps for CTAs 0..n-1.
extern "C" int kp_tc_trace_dump(unsigned long long* out, int n) {
    if (!out || n < 1 || n > kp::tc::TRACE_CTAS) return -1;
    if (cudaMemcpyFromSymbol(out, kp::tc::g_tc_trace, size_t(n) * 16 * sizeof(unsigned long long)) !=
        cudaSuccess)
        return -1;
    return 0;
}
#endif
