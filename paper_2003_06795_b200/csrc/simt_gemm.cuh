// K1: FP32 FFMA register-tiled GEMM family (the paper's 640-point space).
//
// Geometry follows the reference's only executable description of the kernel
// family, synthetic.analytic_perf (reference pkg/src/kernelprune/synthetic.py:
// 65-70):
//   * each thread (work item) owns a row_tile x col_tile block of C,
//   * a work-group of wg_rows x wg_cols threads owns a
//     (row_tile*wg_rows) x (col_tile*wg_cols) block of C,
//   * K is consumed `acc` values per register step: a thread loads `acc`
//     k-slices of its A and B fragments, then issues acc*row_tile*col_tile
//     FFMAs ((row_tile+col_tile)*acc fragment registers).
// row_tile/col_tile/acc are template parameters (64 kernels per operand
// layout); the work-group shape is a runtime launch parameter, as in the paper
// ("can be set at runtime and do not require additional kernels").
//
// B200 mapping:
//   * shared memory keeps each operand in its global orientation, K depth
//     BK = 32 (16 for the largest tiles) per stage, 2/3-stage cp.async ring (16-byte copies when rows
//     are 16-byte aligned, zero-filling 4-byte copies otherwise):
//       m/n-contiguous sources (A transposed, B normal): "chunk" layout, 4
//         output rows x BK K-slices per padded chunk (chunk_off); a thread
//         owns 4-wide row chunks strided by 4*wg and reads one LDS.128 per
//         chunk per K slice, and stores C with 16-byte STG;
//       B transposed: transposed into the chunk layout by 4-byte cp.async
//         (copy_transpose), so B fragments are always column vectors;
//       k-contiguous A (A normal): "row" layout (RS
//         pitch); a thread owns rows t + i*wg and reads K vectors of width
//         min(acc, 4) per row -- `acc` is the K vector width, as in the
//         paper's kernel;
//     every fragment address is a per-thread base plus a compile-time offset,
//     and the 8 threads of a quarter-warp always hit 8 distinct bank groups;
//   * every C element accumulates its K products in increasing k with fmaf,
//     starting from +0, so results are bit-identical to the sequential-fmaf
//     oracle (oracle/gemm_ref.c); K/M/N tails are zero-filled in shared memory.
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <map>
#include <type_traits>
#include <mutex>
#include <utility>

#include "kp_internal.cuh"

namespace kp {
namespace simt {

constexpr int GROUP_M = 8;  // tile raster: 8 m-tiles share a sweep over n

// Shared K depth per pipeline stage: 32 when two stages of it fit in 112 KB
// (two CTAs per SM), else 16 -- halves the per-K-slice copy/sync overhead of
// the common tiles without starving the huge (1024-row) ones.
template <int BK>
struct Geo {
    static constexpr int LOG_BK = BK == 32 ? 5 : 4;
    static constexpr int CH = BK * 4 + 4;  // chunk pitch (floats), see chunk_off
    static constexpr int RS = BK + 4;      // row pitch (floats), see copy_rows
};

struct Params {
    const float* A;
    const float* B;
    float* C;
    int M, N, K;
    int64_t lda, ldb, ldc, sa, sb, sc;
    float alpha, beta;
    int wgr, wgc, log_wgc, log_nthr;
    int log_bm, log_bn;
    int stages;
    int vecA, vecB, vecC;
    int tiles_m, tiles_n;
    int a_elems, b_elems;    // floats per stage (chunk-major tiles)
    // ordered stream-K (sk != 0): gridDim.x persistent CTAs share
    // units = tiles*batch*KT (tile, k-slice) units; hand-off flags live in a
    // ring of KP_SK_RING slots owned by the library
    int sk;
    int64_t units, dp_tiles;
    uint32_t* flags;
    uint32_t flag_base, epoch;
};

// Shared-memory tile layout ("chunk-major"): an operand tile of BM (or BN)
// rows of the output axis is stored as BM/4 chunks of 4 consecutive rows, each
// chunk holding its BK K-slices as 16-byte float4s:
//     element (k, m)  at  (m >> 2) * CH + k * 4 + (m & 3),   CH = BK*4 + 4.
// (CH/4 is odd, so 8 consecutive chunks start in 8 distinct bank groups.)
// A thread's 4-row fragment at slice k is one LDS.128 whose offset is a
// per-thread base plus the compile-time k*4, so the unrolled K loop needs no
// address arithmetic (the runtime work-group shape only enters the bases);
// the 4-float pad per chunk makes 8 consecutive chunks hit 8 different 16-byte
// bank groups.
template <int BK>
__device__ __forceinline__ int chunk_off(int k, int m) {
    return (m >> 2) * Geo<BK>::CH + k * 4 + (m & 3);
}

// Copy a BK x cols block whose rows are K and whose columns (the M/N axis,
// cols = 1 << log_cols) are contiguous in global memory (element (k, c) at
// src[k*ld + c]) into the chunk-major tile at shared address `s`. Elements
// with k >= kv or c >= cv are written as zero. 16-byte copies when vec.
template <int BK>
__device__ __forceinline__ void copy_direct(uint32_t s, const float* src, int64_t ld, int log_cols,
                                            int cv, int kv, bool vec, int tid, int nthr) {
    if (vec && log_cols >= 2) {
        const int log_cpr = log_cols - 2;
        const int total = BK << log_cpr;
        if ((nthr >> log_cpr) > 0 && total <= 8 * nthr) {
            // fast: every chunk of this thread sits in one column, dr K-rows apart
            const int r0 = tid >> log_cpr;
            const int c0 = (tid & ((1 << log_cpr) - 1)) << 2;
            const int dr = nthr >> log_cpr;
            const int n = total >= nthr ? total / nthr : (tid < total ? 1 : 0);
            const int cbytes = min(max(cv - c0, 0), 4) * 4;
            const float* gp = src + (int64_t)r0 * ld + c0;
            const int64_t gstep = (int64_t)dr * ld;
            const uint32_t sp = s + 4u * chunk_off<BK>(r0, c0);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                if (c < n) {
                    cp_async16(sp + c * dr * 16, gp, r0 + c * dr < kv ? cbytes : 0);
                    gp += gstep;
                }
            }
            return;
        }
        for (int idx = tid; idx < total; idx += nthr) {
            const int r = idx >> log_cpr;
            const int c = (idx & ((1 << log_cpr) - 1)) << 2;
            cp_async16(s + 4u * chunk_off<BK>(r, c), src + (int64_t)r * ld + c,
                       r < kv ? min(max(cv - c, 0), 4) * 4 : 0);
        }
        return;
    }
    const int total = BK << log_cols;
    for (int idx = tid; idx < total; idx += nthr) {
        const int r = idx >> log_cols;
        const int c = idx & ((1 << log_cols) - 1);
        cp_async4(s + 4u * chunk_off<BK>(r, c), src + (int64_t)r * ld + c, (r < kv && c < cv) ? 4 : 0);
    }
}

// Vector shared-memory load of W consecutive floats (W in 1,2,4).
template <int W>
__device__ __forceinline__ void lds(const float* p, float* out) {
    if constexpr (W == 1) {
        out[0] = p[0];
    } else if constexpr (W == 2) {
        const float2 v = *reinterpret_cast<const float2*>(p);
        out[0] = v.x; out[1] = v.y;
    } else {
        const float4 v = *reinterpret_cast<const float4*>(p);
        out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
    }
}

// Row layout ("R") for k-contiguous sources (A normal, B transposed): the
// tile is stored as global rows, element (k, r) at r*RS + k with RS = BK + 4,
// filled by 16-byte cp.async along k without any transpose. A thread owns
// rows t + i*wg, so the 8 threads of a quarter-warp read 8 consecutive rows
// (20-float pitch -> 8 distinct 16-byte bank groups) and each fragment read is
// a float vector of up to 4 K values of one row.
template <int BK>
__device__ __forceinline__ void copy_rows(uint32_t s, const float* src, int64_t ld, int log_rows,
                                          int rv, int kv, bool vec, int tid, int nthr) {
    constexpr int RS = Geo<BK>::RS, TPR = BK / 4, LOG_TPR = BK == 32 ? 3 : 2;
    const int rows = 1 << log_rows;
    if (vec) {
        const int c0 = (tid & (TPR - 1)) << 2;  // BK/4 threads per row
        const int dr = nthr >> LOG_TPR;
        const int kbytes = min(max(kv - c0, 0), 4) * 4;
        const float* gp = src + (int64_t)(tid >> LOG_TPR) * ld + c0;
        const int64_t gstep = (int64_t)dr * ld;
        for (int r = tid >> LOG_TPR; r < rows; r += dr) {
            cp_async16(s + 4u * (r * RS + c0), gp, r < rv ? kbytes : 0);
            gp += gstep;
        }
        return;
    }
    const int total = rows << Geo<BK>::LOG_BK;
    for (int idx = tid; idx < total; idx += nthr) {
        const int r = idx >> Geo<BK>::LOG_BK;
        const int c = idx & (BK - 1);
        cp_async4(s + 4u * (r * RS + c), src + (int64_t)r * ld + c, (r < rv && c < kv) ? 4 : 0);
    }
}

// Thread t's fragment along one output axis, for a K group of ACC slices.
//   KROW (row layout):  rows t + i*wg, ACC-wide K vectors per row.
//   chunk layout:       T >= 4 -> chunks q*wg + t (rows q*4*wg + t*4 + e),
//                       else rows t*T + i; one T-wide vector per K slice.
// Offsets are per-thread bases; the K offsets are compile-time immediates.
template <bool KROW, int T, int ACC, int BK>
struct Frag {
    static constexpr int CH = Geo<BK>::CH, RS = Geo<BK>::RS;
    static constexpr int NB = KROW ? T : (T >= 4 ? T / 4 : 1);
    int off[NB];

    __device__ __forceinline__ void init(int t, int wg) {
        if constexpr (KROW) {
#pragma unroll
            for (int i = 0; i < T; ++i) off[i] = (t + i * wg) * RS;
        } else if constexpr (T >= 4) {
#pragma unroll
            for (int q = 0; q < T / 4; ++q) off[q] = (q * wg + t) * CH;
        } else {
            off[0] = ((t * T) >> 2) * CH + ((t * T) & 3);
        }
    }
    __device__ __forceinline__ void load(const float* stage, int kb, float (&out)[ACC][T]) const {
        if constexpr (KROW) {
            constexpr int V = ACC < 4 ? ACC : 4;
#pragma unroll
            for (int i = 0; i < T; ++i) {
#pragma unroll
                for (int h = 0; h < ACC / V; ++h) {
                    float v[V];
                    lds<V>(stage + off[i] + kb + h * V, v);
#pragma unroll
                    for (int e = 0; e < V; ++e) out[h * V + e][i] = v[e];
                }
            }
        } else {
#pragma unroll
            for (int kk = 0; kk < ACC; ++kk) {
                if constexpr (T >= 4) {
#pragma unroll
                    for (int q = 0; q < T / 4; ++q)
                        lds<4>(stage + off[q] + (kb + kk) * 4, &out[kk][4 * q]);
                } else {
                    lds<T>(stage + off[0] + (kb + kk) * 4, &out[kk][0]);
                }
            }
        }
    }
    __device__ __forceinline__ static int index(int i, int t, int wg) {
        if constexpr (KROW) return t + i * wg;
        else if constexpr (T >= 4) return (i / 4) * 4 * wg + t * 4 + (i % 4);
        else return t * T + i;
    }
};

// Accumulator tile on Blackwell's packed FP32 pipe (FFMA2, `__ffma2_rn`):
// two C elements share one 64-bit register pair and one instruction updates
// both with the same single-rounding FMA as fmaf, so the increasing-k fmaf
// chain of every element (and bit-exactness vs the oracle) is unchanged while
// the FFMA issue count halves.  When B is staged n-contiguous (chunk layout:
// B normal, or B transposed through copy_transpose) its fragment holds
// adjacent columns in adjacent registers and pairs run along columns;
// otherwise pairs run along rows when A is transposed (chunk layout), and the
// remaining cases (A normal x row-staged B, 1x1 tiles) stay on scalar FFMA --
// pairing values from different loads would cost a move per FFMA2.  The broadcast
// operand costs nothing: ptxas folds make_float2(x, x) into FFMA2's
// scalar-operand form.
template <int RT, int CT, bool TA, bool B_CHUNK>
struct AccTile {
    static constexpr int PAIR = (B_CHUNK && CT >= 2) ? 1 : (TA && RT >= 2) ? 2 : 0;  // 1: column pairs, 2: row pairs
    static constexpr int PR = PAIR == 2 ? RT / 2 : RT;
    static constexpr int PC = PAIR == 1 ? CT / 2 : CT;
    using Elem = typename std::conditional<PAIR == 0, float, float2>::type;
    Elem v[PR][PC];

    __device__ __forceinline__ float& at(int i, int j) {
        if constexpr (PAIR == 1) return (j & 1) ? v[i][j >> 1].y : v[i][j >> 1].x;
        else if constexpr (PAIR == 2) return (i & 1) ? v[i >> 1][j].y : v[i >> 1][j].x;
        else return v[i][j];
    }
    template <int ACC>
    __device__ __forceinline__ void fma(const float (&a)[ACC][RT], const float (&b)[ACC][CT]) {
#pragma unroll
        for (int kk = 0; kk < ACC; ++kk) {
            if constexpr (PAIR == 1) {
#pragma unroll
                for (int i = 0; i < RT; ++i)
#pragma unroll
                    for (int jp = 0; jp < PC; ++jp)
                        v[i][jp] = __ffma2_rn(make_float2(a[kk][i], a[kk][i]),
                                              make_float2(b[kk][2 * jp], b[kk][2 * jp + 1]), v[i][jp]);
            } else if constexpr (PAIR == 2) {
#pragma unroll
                for (int ip = 0; ip < PR; ++ip)
#pragma unroll
                    for (int j = 0; j < CT; ++j)
                        v[ip][j] = __ffma2_rn(make_float2(a[kk][2 * ip], a[kk][2 * ip + 1]),
                                              make_float2(b[kk][j], b[kk][j]), v[ip][j]);
            } else {
#pragma unroll
                for (int i = 0; i < RT; ++i)
#pragma unroll
                    for (int j = 0; j < CT; ++j) v[i][j] = fmaf(a[kk][i], b[kk][j], v[i][j]);
            }
        }
    }
};

__device__ __forceinline__ float epilogue(float acc, float alpha, float beta, const float* c_old) {
    const float v = alpha * acc;
    return beta == 0.0f ? v : fmaf(beta, *c_old, v);
}

// Interior-tile copies (no M/N/K tail, 16-byte aligned rows): fixed 16-byte
// cp.async, the per-thread pointers advance by a constant stride, no zero-fill
// size arithmetic.  Same shared layouts as copy_rows / copy_direct.
template <int BK>
__device__ __forceinline__ void copy_rows_full(uint32_t s, const float* src, int64_t ld,
                                               int log_rows, int tid, int log_nthr) {
    constexpr int RS = Geo<BK>::RS, TPR = BK / 4, LOG_TPR = BK == 32 ? 3 : 2;
    const int r0 = tid >> LOG_TPR, c0 = (tid & (TPR - 1)) << 2;
    const int log_dr = log_nthr - LOG_TPR;
    // rows and dr are powers of two: n = rows/dr copies, or one for r0 < rows
    const int n = log_rows >= log_dr ? 1 << (log_rows - log_dr) : int(r0 < (1 << log_rows));
    const float* gp = src + (int64_t)r0 * ld + c0;
    uint32_t sp = s + 4u * (r0 * RS + c0);
    const int64_t gstep = ld << log_dr;
    const uint32_t sstep = (4u * RS) << log_dr;
#pragma unroll 2
    for (int i = 0; i < n; ++i) {
        cp_async16_full(sp, gp);
        gp += gstep;
        sp += sstep;
    }
}

template <int BK>
__device__ __forceinline__ void copy_direct_full(uint32_t s, const float* src, int64_t ld,
                                                 int log_cols, int tid, int log_nthr) {
    const int log_cpr = log_cols - 2;  // float4s per K row
    if (log_nthr >= log_cpr) {  // every copy of this thread sits in one column, dr K-rows apart
        const int log_dr = log_nthr - log_cpr;
        const int r0 = tid >> log_cpr, c0 = (tid & ((1 << log_cpr) - 1)) << 2;
        const int n = Geo<BK>::LOG_BK >= log_dr ? 1 << (Geo<BK>::LOG_BK - log_dr) : int(r0 < BK);
        const float* gp = src + (int64_t)r0 * ld + c0;
        uint32_t sp = s + 4u * chunk_off<BK>(r0, c0);
        const int64_t gstep = ld << log_dr;
        const uint32_t sstep = 16u << log_dr;
#pragma unroll 2
        for (int i = 0; i < n; ++i) {
            cp_async16_full(sp, gp);
            gp += gstep;
            sp += sstep;
        }
        return;
    }
    // wide tiles: more float4s per K row than threads
    const int total = BK << log_cpr, nthr = 1 << log_nthr;
    for (int idx = tid; idx < total; idx += nthr) {
        const int r = idx >> log_cpr;
        const int c = (idx & ((1 << log_cpr) - 1)) << 2;
        cp_async16_full(s + 4u * chunk_off<BK>(r, c), src + (int64_t)r * ld + c);
    }
}

// B stored n x k (k contiguous, B transposed), staged transposed into the
// chunk layout, so the B fragment is one LDS.128 of 4 adjacent columns per k
// (FFMA2 column pairs, 16-byte C stores) whatever the operand layout.  4-byte
// cp.async; consecutive threads take (n & 3) fastest, then k: a warp reads 4
// rows x 8 consecutive k (whole 32-byte sectors) and writes 32 consecutive
// shared words (no bank conflict).  Elements with n >= rv or k >= kv are
// zero-filled unless `full`.
template <int BK>
__device__ __forceinline__ void copy_transpose(uint32_t s, const float* src, int64_t ld,
                                               int log_rows, int rv, int kv, bool full, int tid,
                                               int log_nthr) {
    constexpr int LOG_BK = Geo<BK>::LOG_BK;
    const int rows = 1 << log_rows;
    if (log_rows >= 2 && log_nthr >= LOG_BK + 2) {  // (k, n & 3) fixed per thread
        const int nl = tid & 3, k = (tid >> 2) & (BK - 1);
        const int dn = 1 << (log_nthr - LOG_BK);     // rows advanced per copy (multiple of 4)
        const int n0 = ((tid >> (LOG_BK + 2)) << 2) + nl;
        const float* gp = src + (int64_t)n0 * ld + k;
        uint32_t sp = s + 4u * chunk_off<BK>(k, n0);
        const int64_t gstep = (int64_t)dn * ld;
        const uint32_t sstep = 4u * (dn >> 2) * Geo<BK>::CH;
        if (full) {
#pragma unroll 4
            for (int n = n0; n < rows; n += dn) {
                cp_async4_full(sp, gp);
                gp += gstep;
                sp += sstep;
            }
        } else {
            for (int n = n0; n < rows; n += dn) {
                cp_async4(sp, gp, (n < rv && k < kv) ? 4 : 0);
                gp += gstep;
                sp += sstep;
            }
        }
        return;
    }
    const int lr = log_rows < 2 ? log_rows : 2;  // low bits of n taken fastest
    const int total = rows << LOG_BK, nthr = 1 << log_nthr;
    for (int idx = tid; idx < total; idx += nthr) {
        const int k = (idx >> lr) & (BK - 1);
        const int n = ((idx >> (lr + LOG_BK)) << lr) + (idx & ((1 << lr) - 1));
        cp_async4(s + 4u * chunk_off<BK>(k, n), src + (int64_t)n * ld + k,
                  (full || (n < rv && k < kv)) ? 4 : 0);
    }
}

// Interior copy plan, hoisted out of the K loop (round 2).  The *_full copies
// above rebuild every pointer, shift and trip count from the kernel
// parameters at each K slice -- ~220 non-FMA instructions per warp per slice
// in the selected 2048^3 kernel, issued as one dependent burst right after
// the barrier.  For a tile whose copies all take the interior path, the
// per-thread part (first global source, shared offset within a stage, copies
// per slice) is computed once per tile; a slice is then n copies along two
// constant strides plus one pointer bump.  Same element -> shared-address
// mapping as copy_rows_full / copy_direct_full / copy_transpose(full), so
// the staged tiles (and every result bit) are unchanged.
struct CopyPlan {
    const float* gp;  // this thread's first source element at the next slice
    uint32_t sp;      // byte offset of its first destination within a stage
    int n;            // copies per slice
    int64_t gstep;    // global element stride between this thread's copies
    uint32_t sstep;   // shared byte stride between them
    int64_t kstep;    // global element advance per K slice
};

// k-contiguous source (A normal, B transposed kept as rows): copy_rows_full.
template <int BK>
__device__ __forceinline__ CopyPlan plan_rows(const float* src, int64_t ld, int log_rows, int tid,
                                              int log_nthr) {
    constexpr int RS = Geo<BK>::RS, TPR = BK / 4, LOG_TPR = BK == 32 ? 3 : 2;
    const int r0 = tid >> LOG_TPR, c0 = (tid & (TPR - 1)) << 2;
    const int log_dr = log_nthr - LOG_TPR;
    CopyPlan c;
    c.n = log_rows >= log_dr ? 1 << (log_rows - log_dr) : int(r0 < (1 << log_rows));
    c.gp = src + (int64_t)r0 * ld + c0;
    c.sp = 4u * (r0 * RS + c0);
    c.gstep = ld << log_dr;
    c.sstep = (4u * RS) << log_dr;
    c.kstep = BK;
    return c;
}

// K-row source (A transposed, B normal), chunk layout: copy_direct_full's
// one-column-per-thread case (the caller checks log_nthr >= log_cols - 2).
template <int BK>
__device__ __forceinline__ CopyPlan plan_direct(const float* src, int64_t ld, int log_cols, int tid,
                                                int log_nthr) {
    const int log_cpr = log_cols - 2;
    const int log_dr = log_nthr - log_cpr;
    const int r0 = tid >> log_cpr, c0 = (tid & ((1 << log_cpr) - 1)) << 2;
    CopyPlan c;
    c.n = Geo<BK>::LOG_BK >= log_dr ? 1 << (Geo<BK>::LOG_BK - log_dr) : int(r0 < BK);
    c.gp = src + (int64_t)r0 * ld + c0;
    c.sp = 4u * chunk_off<BK>(r0, c0);
    c.gstep = ld << log_dr;
    c.sstep = 16u << log_dr;
    c.kstep = (int64_t)BK * ld;
    return c;
}

// B transposed, staged transposed (4-byte copies): copy_transpose's
// fixed-(k, n & 3) case (the caller checks log_rows >= 2, log_nthr >= LOG_BK + 2).
template <int BK>
__device__ __forceinline__ CopyPlan plan_transpose(const float* src, int64_t ld, int log_rows,
                                                   int tid, int log_nthr) {
    constexpr int LOG_BK = Geo<BK>::LOG_BK;
    const int nl = tid & 3, k = (tid >> 2) & (BK - 1);
    const int dn = 1 << (log_nthr - LOG_BK);
    const int n0 = ((tid >> (LOG_BK + 2)) << 2) + nl;
    const int rows = 1 << log_rows;
    CopyPlan c;
    c.n = n0 < rows ? (rows - n0 + dn - 1) / dn : 0;
    c.gp = src + (int64_t)n0 * ld + k;
    c.sp = 4u * chunk_off<BK>(k, n0);
    c.gstep = (int64_t)dn * ld;
    c.sstep = 4u * (dn >> 2) * Geo<BK>::CH;
    c.kstep = BK;
    return c;
}

// One slice of a plan into the stage at shared byte address `s`; advances
// the plan to the next slice.
template <bool FOUR_BYTE>
__device__ __forceinline__ void plan_issue(CopyPlan& c, uint32_t s) {
    const float* gp = c.gp;
    uint32_t sp = s + c.sp;
#pragma unroll 2
    for (int i = 0; i < c.n; ++i) {
        if constexpr (FOUR_BYTE) cp_async4_full(sp, gp);
        else cp_async16_full(sp, gp);
        gp += c.gstep;
        sp += c.sstep;
    }
    c.gp += c.kstep;
}

// Ordered stream-K hand-off.  A tile split between CTAs c and c+1 is computed
// k-slices [0, j) by c and [j, KT) by c+1; c writes its raw accumulators into
// the C tile (beta == 0, so C is scratch until its final write) and publishes
// `epoch` in its flag; c+1 starts from those accumulators.  The fmaf order of
// every C element is therefore the same increasing-k chain as the one-CTA
// kernel (bit-identical results).
__device__ __forceinline__ void flag_publish(uint32_t* flag, uint32_t epoch) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;\n" :: "l"(flag), "r"(epoch) : "memory");
}
__device__ __forceinline__ void flag_wait(const uint32_t* flag, uint32_t epoch) {
    const long long t0 = clock64();
    while (true) {
        uint32_t v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(flag) : "memory");
        if (v == epoch) return;
        if (clock64() - t0 > (1LL << 34)) __trap();  // ~9 s: never hang the GPU
        __nanosleep(64);
    }
}

// BT (B transposed only): stage B transposed into the chunk layout (true) or
// keep its k-contiguous rows (false); chosen per problem by launch().
template <int ACC, int RT, int CT, bool TA, bool TB, int BK, bool BT>
#ifndef KP_SIMT_MIN_BLOCKS
#define KP_SIMT_MIN_BLOCKS 2
#endif
__global__ void __launch_bounds__(256, KP_SIMT_MIN_BLOCKS) simt_gemm_kernel(const Params p) {
    constexpr int LOG_BK = Geo<BK>::LOG_BK;
    extern __shared__ __align__(16) float smem[];
    const int tid = threadIdx.x;
    const int nthr = p.wgr * p.wgc;
    const int ty = tid >> p.log_wgc;
    const int tx = tid & (p.wgc - 1);
    const int bm = 1 << p.log_bm, bn = 1 << p.log_bn;

    float* sA = smem;
    float* sB = smem + p.stages * p.a_elems;
    const uint32_t sA_u = smem_u32(sA), sB_u = smem_u32(sB);
    const int KT = (p.K + BK - 1) >> LOG_BK;
    const int tiles = p.tiles_m * p.tiles_n;

    // ---- schedule: which (tile, k-slice range) segments this CTA computes.
    // Classic: one whole tile per CTA (blockIdx.z = batch).  Ordered stream-K:
    // CTA c owns units [c*U/G, (c+1)*U/G) of the U = tiles*batch*KT
    // (tile, k-slice) units; it first computes the leading k-slices of its
    // last tile (hand-off to c+1), then its whole tiles, then the trailing
    // k-slices of its first tile (hand-off from c-1, published long before).
    int64_t full_lo, full_hi, st_tile = -1, fin_tile = -1;
    int st_ke = 0, fin_kb = 0, n_dp = 0;
    if (!p.sk) {
        full_lo = (int64_t)blockIdx.z * tiles + blockIdx.x;
        full_hi = full_lo + 1;
    } else {
        // whole waves first (tiles c, c+G, ... below dp_tiles: neighbouring CTAs
        // on neighbouring tiles), then the stream-K region of 1-2 waves
        const int64_t G = gridDim.x, c = blockIdx.x;
        n_dp = int(p.dp_tiles / G);
        const int64_t U = p.units - p.dp_tiles * KT;
        const int64_t u0 = p.dp_tiles * KT + c * U / G, u1 = p.dp_tiles * KT + (c + 1) * U / G;
        const int64_t tf = u0 / KT, tl = (u1 - 1) / KT;
        const int kf = int(u0 - tf * KT), ke = int(u1 - tl * KT);
        full_lo = kf ? tf + 1 : tf;
        full_hi = ke < KT ? tl : tl + 1;
        if (ke < KT) { st_tile = tl; st_ke = ke; }
        if (kf) { fin_tile = tf; fin_kb = kf; }
    }
    const int nsteps = n_dp + int(st_tile >= 0) + int(full_hi - full_lo) + int(fin_tile >= 0);

    using FragA = Frag<!TA, RT, ACC, BK>;
    constexpr bool B_CHUNK = !TB || BT;  // B staged n-contiguous
    using FragB = Frag<!B_CHUNK, CT, ACC, BK>;
    FragA fa;
    FragB fb;
    fa.init(ty, p.wgr);
    fb.init(tx, p.wgc);
    const int S = p.stages;

    for (int step = 0; step < nsteps; ++step) {
        int64_t T;
        int kb = 0, kend = KT, mode = 0;  // mode 0 whole tile, 1 hand-off out, 2 hand-off in
        const int sks = step - n_dp;      // step within the stream-K region
        if (sks < 0) {
            T = blockIdx.x + (int64_t)step * gridDim.x;
        } else if (st_tile >= 0 && sks == 0) {
            T = st_tile; kend = st_ke; mode = 1;
        } else if (fin_tile >= 0 && step == nsteps - 1) {
            T = fin_tile; kb = fin_kb; mode = 2;
        } else {
            T = full_lo + sks - int(st_tile >= 0);
        }
        const int64_t bz = T / tiles;
        const int tile = int(T - bz * tiles);
        // grouped raster over (tiles_m x tiles_n) for L2 reuse of A rows / B cols
        const int per_group = GROUP_M * p.tiles_n;
        const int group = tile / per_group;
        const int first_m = group * GROUP_M;
        const int gsz = min(p.tiles_m - first_m, GROUP_M);
        const int in_group = tile - group * per_group;
        const int m0 = (first_m + in_group % gsz) << p.log_bm;
        const int n0 = (in_group / gsz) << p.log_bn;
        const float* __restrict__ A = p.A + bz * p.sa;
        const float* __restrict__ B = p.B + bz * p.sb;
        float* __restrict__ C = p.C + bz * p.sc;
        const bool fullA = p.vecA && m0 + bm <= p.M;
        const bool fullB = p.vecB && n0 + bn <= p.N;

        // hoisted interior plans (see CopyPlan), positioned at slice kb.
        // Thread tiles up to 32 outputs only: the 8x8 tiles already sit at
        // the 128-register cap, where the plan's ~10 live registers cost more
        // than the copy arithmetic it removes (profiles/k1_ab/ab_hoist_*.jsonl:
        // 8x8 NN/NT -4..-9 %, <= 32-output tiles +0..+7 %).
        constexpr bool HOIST = RT * CT <= 32;
        const int64_t kb0 = (int64_t)kb << LOG_BK;
        bool planA_ok = false, planB_ok = false;
        CopyPlan pa{}, pb{};
        if constexpr (!HOIST) {
        } else if constexpr (TA) {
            planA_ok = fullA && p.log_nthr >= p.log_bm - 2;
            pa = plan_direct<BK>(A + kb0 * p.lda + m0, p.lda, p.log_bm, tid, p.log_nthr);
        } else {
            planA_ok = fullA;
            pa = plan_rows<BK>(A + (int64_t)m0 * p.lda + kb0, p.lda, p.log_bm, tid, p.log_nthr);
        }
        if constexpr (!HOIST) {
        } else if constexpr (!TB) {
            planB_ok = fullB && p.log_nthr >= p.log_bn - 2;
            pb = plan_direct<BK>(B + kb0 * p.ldb + n0, p.ldb, p.log_bn, tid, p.log_nthr);
        } else if constexpr (BT) {
            planB_ok = n0 + bn <= p.N && p.log_bn >= 2 && p.log_nthr >= LOG_BK + 2;
            pb = plan_transpose<BK>(B + (int64_t)n0 * p.ldb + kb0, p.ldb, p.log_bn, tid, p.log_nthr);
        } else {
            planB_ok = fullB;
            pb = plan_rows<BK>(B + (int64_t)n0 * p.ldb + kb0, p.ldb, p.log_bn, tid, p.log_nthr);
        }

        auto issue = [&](int kt, int stage) {
            const int k0 = kt << LOG_BK;
            const uint32_t a_dst = sA_u + 4u * stage * p.a_elems;
            const uint32_t b_dst = sB_u + 4u * stage * p.b_elems;
            const bool kfull = k0 + BK <= p.K;
            // slices are issued in increasing kt from kb, so the plans'
            // running pointers sit at kt whenever the interior path is taken
            // (only the last slice of a ragged K can leave it)
            if (HOIST && kfull && planA_ok && planB_ok) {
                plan_issue<false>(pa, a_dst);
                plan_issue<TB && BT>(pb, b_dst);
                return;
            }
            if constexpr (TA) {  // A stored k x m: rows are K
                const float* src = A + (int64_t)k0 * p.lda + m0;
                if (fullA && kfull) copy_direct_full<BK>(a_dst, src, p.lda, p.log_bm, tid, p.log_nthr);
                else copy_direct<BK>(a_dst, src, p.lda, p.log_bm, p.M - m0, p.K - k0, p.vecA, tid, nthr);
            } else {             // A stored m x k: k-contiguous rows, row layout
                const float* src = A + (int64_t)m0 * p.lda + k0;
                if (fullA && kfull) copy_rows_full<BK>(a_dst, src, p.lda, p.log_bm, tid, p.log_nthr);
                else copy_rows<BK>(a_dst, src, p.lda, p.log_bm, p.M - m0, p.K - k0, p.vecA, tid, nthr);
            }
            if constexpr (!TB) { // B stored k x n: rows are K
                const float* src = B + (int64_t)k0 * p.ldb + n0;
                if (fullB && kfull) copy_direct_full<BK>(b_dst, src, p.ldb, p.log_bn, tid, p.log_nthr);
                else copy_direct<BK>(b_dst, src, p.ldb, p.log_bn, p.N - n0, p.K - k0, p.vecB, tid, nthr);
            } else if constexpr (BT) {  // B stored n x k, transposed into the chunk layout
                copy_transpose<BK>(b_dst, B + (int64_t)n0 * p.ldb + k0, p.ldb, p.log_bn, p.N - n0,
                                   p.K - k0, n0 + bn <= p.N && kfull, tid, p.log_nthr);
            } else {             // B stored n x k: k-contiguous rows, row layout
                const float* src = B + (int64_t)n0 * p.ldb + k0;
                if (fullB && kfull) copy_rows_full<BK>(b_dst, src, p.ldb, p.log_bn, tid, p.log_nthr);
                else copy_rows<BK>(b_dst, src, p.ldb, p.log_bn, p.N - n0, p.K - k0, p.vecB, tid, nthr);
            }
        };

        if (step > 0) __syncthreads();  // every warp is done reading the previous segment's stages
        for (int s = 0; s < S - 1; ++s) {
            if (kb + s < kend) issue(kb + s, s);
            cp_async_commit();
        }

        AccTile<RT, CT, TA, B_CHUNK> acc;
        if (mode == 2) {  // continue the k chain of CTA blockIdx.x - 1
            if (tid == 0) flag_wait(p.flags + ((p.flag_base + blockIdx.x - 1) & KP_SK_RING_MASK), p.epoch);
            __syncthreads();
#pragma unroll
            for (int i = 0; i < RT; ++i) {
                const int m = m0 + FragA::index(i, ty, p.wgr);
#pragma unroll
                for (int j = 0; j < CT; ++j) {
                    const int n = n0 + FragB::index(j, tx, p.wgc);
                    acc.at(i, j) = (m < p.M && n < p.N) ? __ldcg(C + (int64_t)m * p.ldc + n) : 0.0f;
                }
            }
        } else {
#pragma unroll
            for (int i = 0; i < RT; ++i)
#pragma unroll
                for (int j = 0; j < CT; ++j) acc.at(i, j) = 0.0f;
        }

        int rd = 0, wr = S - 1;  // stage being read / written
        for (int kt = kb; kt < kend; ++kt) {
            if (S == 3) cp_async_wait<1>(); else cp_async_wait<0>();
            __syncthreads();
            if (kt + S - 1 < kend) issue(kt + S - 1, wr);
            cp_async_commit();
            wr = (wr + 1 == S) ? 0 : wr + 1;
            const float* a_s = sA + rd * p.a_elems;
            const float* b_s = sB + rd * p.b_elems;
            rd = (rd + 1 == S) ? 0 : rd + 1;
#pragma unroll
            for (int kq = 0; kq < BK; kq += ACC) {
                float a[ACC][RT];
                float b[ACC][CT];
                fa.load(a_s, kq, a);
                fb.load(b_s, kq, b);
                acc.template fma<ACC>(a, b);
            }
        }
        cp_async_wait<0>();

        // epilogue: C = alpha*acc (+ beta*C); a hand-off stores the raw chain
        const float alpha = mode == 1 ? 1.0f : p.alpha;
        const float beta = mode == 1 ? 0.0f : p.beta;
#pragma unroll
        for (int i = 0; i < RT; ++i) {
            const int m = m0 + FragA::index(i, ty, p.wgr);
            if (m >= p.M) continue;
            float* crow = C + (int64_t)m * p.ldc;
            if constexpr (B_CHUNK && CT >= 4) {
#pragma unroll
                for (int q = 0; q < CT / 4; ++q) {
                    const int n = n0 + q * 4 * p.wgc + tx * 4;
                    if (p.vecC && n + 3 < p.N) {
                        float4 v;
                        if (beta == 0.0f) {
                            v = make_float4(alpha * acc.at(i, 4 * q), alpha * acc.at(i, 4 * q + 1),
                                            alpha * acc.at(i, 4 * q + 2), alpha * acc.at(i, 4 * q + 3));
                        } else {
                            const float4 o = *reinterpret_cast<const float4*>(crow + n);
                            v = make_float4(fmaf(beta, o.x, alpha * acc.at(i, 4 * q)),
                                            fmaf(beta, o.y, alpha * acc.at(i, 4 * q + 1)),
                                            fmaf(beta, o.z, alpha * acc.at(i, 4 * q + 2)),
                                            fmaf(beta, o.w, alpha * acc.at(i, 4 * q + 3)));
                        }
                        *reinterpret_cast<float4*>(crow + n) = v;
                    } else {
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            if (n + e < p.N)
                                crow[n + e] = epilogue(acc.at(i, 4 * q + e), alpha, beta, crow + n + e);
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < CT; ++j) {
                    const int n = n0 + FragB::index(j, tx, p.wgc);
                    if (n < p.N) crow[n] = epilogue(acc.at(i, j), alpha, beta, crow + n);
                }
            }
        }
        if (mode == 1) {  // publish the partial chain to CTA blockIdx.x + 1
            __threadfence();
            __syncthreads();
            if (tid == 0) flag_publish(p.flags + ((p.flag_base + blockIdx.x) & KP_SK_RING_MASK), p.epoch);
        }
    }
}

inline int ilog2(int v) {
    int l = 0;
    while ((1 << l) < v) ++l;
    return l;
}
inline int round4(int v) { return (v + 3) & ~3; }

// Shared-memory plan for one tile shape: K depth, stage count, bytes.
struct SmemPlan {
    int bk, a_elems, b_elems, stages;
    size_t bytes;
};

inline SmemPlan plan_smem(bool a_rows, bool b_rows, int bm, int bn) {
    auto make = [&](int bk) {
        SmemPlan s;
        s.bk = bk;
        s.a_elems = a_rows ? bm * (bk + 4) : (round4(bm) / 4) * (bk * 4 + 4);
        s.b_elems = b_rows ? bn * (bk + 4) : (round4(bn) / 4) * (bk * 4 + 4);
        const size_t stage = 4u * size_t(s.a_elems + s.b_elems);
        s.stages = (3 * stage <= 112 * 1024) ? 3 : 2;
        s.bytes = s.stages * stage;
        return s;
    };
    const SmemPlan deep = make(32);
    if (deep.bytes <= 112 * 1024) return deep;
    return make(16);
}

template <int ACC, int RT, int CT, bool TA, bool TB>
kp_status launch(const GemmProblem& g, int wgr, int wgc, cudaStream_t stream) {
    const int bm = RT * wgr, bn = CT * wgc;
    // B transposed: stage it transposed (FFMA2 column pairs, 4-byte copies)
    // only for tall problems; measured on the network+squares NT sweep, the
    // transposing copy wins +11 % geomean at m >= 4096, breaks even at
    // 1024-4095 and loses 4-9 % below (copy-bound, small m).
    const bool bt = TB && g.m >= 2048;
    SmemPlan sp = plan_smem(!TA, TB && !bt, bm, bn);
    if (sp.bytes > 227 * 1024) return fail(KP_ERR_UNSUPPORTED, "simt: shared-memory plan too large");
    void (*kern)(const Params) = sp.bk == 32 ? simt_gemm_kernel<ACC, RT, CT, TA, TB, 32, false>
                                             : simt_gemm_kernel<ACC, RT, CT, TA, TB, 16, false>;
    if constexpr (TB) {
        if (bt) kern = sp.bk == 32 ? simt_gemm_kernel<ACC, RT, CT, TA, TB, 32, true>
                                   : simt_gemm_kernel<ACC, RT, CT, TA, TB, 16, true>;
    }
    // per-device opt-in to > 48 KB of dynamic shared memory, register count per kernel
    static std::atomic<uint64_t> attr_set[2][2] = {};
    static int regs[2][2] = {{0, 0}, {0, 0}};
    const uint64_t dev_bit = uint64_t(1) << (current_device() & 63);
    if (!(attr_set[sp.bk == 32][bt].load(std::memory_order_acquire) & dev_bit)) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess)
            return check_launch("cudaFuncSetAttribute");
        cudaFuncAttributes fa;
        if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess) return check_launch("cudaFuncGetAttributes");
        regs[sp.bk == 32][bt] = fa.numRegs > 0 ? fa.numRegs : 128;
        attr_set[sp.bk == 32][bt].fetch_or(dev_bit, std::memory_order_release);
    }
    // A third cp.async stage only if it does not cost resident CTAs: small
    // work-groups are register-limited to 4+ CTAs per SM, where 3 stages of
    // shared memory would cap them at 3 (KP_STAGE_OCC=0: always 3 when they
    // fit in 112 KB, tuning experiments only).
    static const bool stage_occ = [] {
        const char* e = std::getenv("KP_STAGE_OCC");
        return !(e && e[0] == '0');
    }();
    if (stage_occ && sp.stages == 3) {
        const int nthr = wgr * wgc;
        const int warp_regs = ((regs[sp.bk == 32][bt] * 32 + 255) / 256) * 256;
        const int occ_regs = std::min(65536 / (warp_regs * ((nthr + 31) / 32)), 32);
        const size_t smem_sm = 228 * 1024, stage_bytes = sp.bytes / 3;
        const int occ3 = std::min<int>(occ_regs, int(smem_sm / (3 * stage_bytes + 1024)));
        const int occ2 = std::min<int>(occ_regs, int(smem_sm / (2 * stage_bytes + 1024)));
        if (occ2 > occ3) {
            sp.stages = 2;
            sp.bytes = 2 * stage_bytes;
        }
    }
    Params p;
    p.A = static_cast<const float*>(g.A);
    p.B = static_cast<const float*>(g.B);
    p.C = g.C;
    p.M = int(g.m); p.N = int(g.n); p.K = int(g.k);
    p.lda = g.lda; p.ldb = g.ldb; p.ldc = g.ldc;
    p.sa = g.sa; p.sb = g.sb; p.sc = g.sc;
    p.alpha = g.alpha; p.beta = g.beta;
    p.wgr = wgr; p.wgc = wgc; p.log_wgc = ilog2(wgc); p.log_nthr = ilog2(wgr * wgc);
    p.log_bm = ilog2(bm); p.log_bn = ilog2(bn);
    p.stages = sp.stages;
    const bool multi = g.batch > 1;
    // 16-byte copies need 16-byte aligned rows (and a 4-aligned tile extent for
    // the chunk layout of m/n-contiguous operands)
    p.vecA = aligned16(g.A) && g.lda % 4 == 0 && (!multi || g.sa % 4 == 0) && (!TA || bm % 4 == 0);
    p.vecB = aligned16(g.B) && g.ldb % 4 == 0 && (!multi || g.sb % 4 == 0) && (TB || bn % 4 == 0);
    p.vecC = aligned16(g.C) && g.ldc % 4 == 0 && (!multi || g.sc % 4 == 0);
    p.tiles_m = int((g.m + bm - 1) / bm);
    p.tiles_n = int((g.n + bn - 1) / bn);
    p.a_elems = sp.a_elems; p.b_elems = sp.b_elems;
    const int64_t tiles = int64_t(p.tiles_m) * p.tiles_n;
    if (tiles > 0x7fffffffLL || g.batch > 65535)
        return fail(KP_ERR_BAD_SHAPE, "simt: grid too large for this work-group tile");
    const int nthr = wgr * wgc;
    p.sk = 0; p.units = 0; p.dp_tiles = 0; p.flags = nullptr; p.flag_base = 0; p.epoch = 0;
    dim3 grid(unsigned(tiles), 1, unsigned(g.batch));
    // Ordered stream-K (see simt_gemm_kernel): spread the tile x k-slice
    // units evenly over one persistent wave when whole tiles would leave part
    // of the last wave idle.  beta == 0 only (C doubles as the hand-off
    // buffer); at least one k-slice range per CTA, so a tile is split between
    // at most two CTAs and no CTA waits on a chain.
    int sched = simt_schedule();
    // A CUDA-graph capture would bake one flag epoch into every replay (the
    // waiter would see its own epoch from the previous replay): captured
    // launches always take one tile per CTA.
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (sched != 0 && cudaStreamIsCapturing(stream, &cap) == cudaSuccess &&
        cap != cudaStreamCaptureStatusNone)
        sched = 0;
    const int64_t T = tiles * g.batch;
    const int64_t KT = (g.k + sp.bk - 1) / sp.bk;
    if (sched != 0 && g.beta == 0.0f && T >= 2 && KT >= 2 && T * KT < (int64_t(1) << 40)) {
        static std::mutex mu;
        static std::map<std::pair<int, size_t>, int> occ_cache;
        int occ = 0;
        {
            std::lock_guard<std::mutex> lock(mu);
            auto it = occ_cache.find({nthr * 2 + int(bt), sp.bytes});
            if (it == occ_cache.end()) {
                if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nthr, sp.bytes) != cudaSuccess)
                    return check_launch("cudaOccupancyMaxActiveBlocksPerMultiprocessor");
                occ_cache[{nthr * 2 + int(bt), sp.bytes}] = occ;
            } else {
                occ = it->second;
            }
        }
        // KP_SK_OCC (tuning experiments only): cap the stream-K CTAs per SM
        static const int occ_cap = [] {
            const char* e = std::getenv("KP_SK_OCC");
            return e ? std::atoi(e) : 0;
        }();
        if (occ_cap > 0 && occ > occ_cap) occ = occ_cap;
        const int64_t slots = int64_t(sm_count()) * occ;
        int64_t G = 0, dp = 0;
        if (sched == 2) {
            G = std::min(slots, T - 1);
        } else if (T > slots && T < 2 * slots && occ <= 2) {
            // Measured policy (tools/k1_ab.py, profiles/): pays only for a
            // ragged second wave of big (>= 256-thread, <= 2 per SM) CTAs;
            // with more waves, or smaller CTAs, the hardware's own refill of
            // the SMs that finish early already balances the tail.
            if (double(T) / double(2 * slots) < 0.95) G = slots;
        }
        if (G >= 1 && slots >= 1) {
            SkFlags f;
            kp_status st = sk_reserve(uint32_t(G), &f);
            if (st != KP_OK) return st;
            p.sk = 1; p.units = T * KT; p.dp_tiles = dp; p.flags = f.flags; p.flag_base = f.base; p.epoch = f.epoch;
            grid = dim3(unsigned(G), 1, 1);
        }
    }
    kern<<<grid, nthr, sp.bytes, stream>>>(p);
    note_launch();
    return check_launch("simt_gemm_kernel");
}

}  // namespace simt
}  // namespace kp
