// Small-M path ("skinny" GEMM): C = alpha * op(A) @ op(B) + beta * C for
// m <= 16 -- the fully connected layers at batch 1-16 (VGG16 FC6
// 1 x 25088 x 4096, FC7, ResNet-50 / MobileNetV2 FC; the paper's FC dataset
// source).  Such a GEMM reads B (k x n) exactly once and
// everything else is noise: it is HBM bound (fp32, m = 1: 0.5 flop/B), so the
// kernel is built around streaming B at full bandwidth, not around the
// paper's register tile (whose 128-row work-group tiles leave 15/16 of every
// tile empty at m = 1 and give such shapes a handful of CTAs).
//
// Work split: every CTA owns one column block of C and one contiguous K
// range [kb, ke) of one batch; it stages op(A)[0:m, kb:ke) in shared memory
// (fp32) once, then streams its B block with 16-byte non-caching loads.
//   B normal   (k x n, n contiguous): a lane owns VEC adjacent columns, the
//              8 warps take interleaved groups of RPW k-rows (RPW loads in
//              flight per thread); partial sums are reduced across the warps
//              through shared memory in warp order 0..7.
//   B transposed (n x k, k contiguous): a warp owns NCW columns, its lanes
//              split K in VEC-wide vectors; partial sums are reduced across
//              the lanes with a warp-shuffle butterfly.
// K ranges: when the column blocks alone cannot fill the GPU, K is split into
// S ranges; each range writes an fp32 partial block to a per-device
// workspace and the CTA that finishes a column block last sums its S
// partials in split order 0..S-1, then applies alpha / beta.  Every
// summation order is fixed by the launch geometry, so results are
// run-to-run deterministic; they are not the sequential-fmaf order of the
// K1 oracle, so parity is checked against the fp64 oracle within the
// K-scaled bound (tests/test_skinny_gpu.py).
// Inputs: fp32 (KP_F32_SIMT and KP_TF32_TC: full fp32 products, at least as
// accurate as TF32) or bf16 (KP_BF16_TC); accumulation is fp32 FMA.
#include <cuda_bf16.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <utility>
#include <vector>

#include "kp_internal.cuh"
#include "skinny_registry.h"

namespace kp {
namespace skinny {

constexpr int THREADS = 256;
constexpr int WARPS = THREADS / 32;
constexpr int MAX_SMEM = 64 * 1024;  // A slice / warp partials: 3 CTAs per SM

struct SkParams {
    const void* A;
    const void* B;
    float* C;
    float* ws;       // split partials [split][batch][m][n] (splits > 1)
    unsigned* counters;  // per (batch, column block) arrival counters (splits > 1)
    int m, n, k;
    int ta;
    int64_t lda, ldb, ldc, sa, sb, sc;
    float alpha, beta;
    int splits, kr;  // K ranges and rows per range
    int batch;
    int groups;      // B transposed: column groups per CTA (reuse of the staged A slice)
};

// ---------------------------------------------------------- element loads
template <typename T>
__device__ __forceinline__ float to_f(T x);
template <>
__device__ __forceinline__ float to_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

// VEC consecutive elements of T starting at p (16- or 8-byte aligned when
// VEC * sizeof(T) >= 8): streamed once, so the load bypasses L1 allocation.
// The raw 32-bit words stay packed in registers (two bf16 per word) and are
// widened to fp32 only when used.
template <typename T, int VEC>
struct Vec {
    static constexpr int BYTES = VEC * int(sizeof(T));
    static constexpr bool RAW = BYTES >= 8;
    static constexpr int WORDS = RAW ? BYTES / 4 : VEC;
    uint32_t w[WORDS];
    __device__ __forceinline__ void load(const T* p) {
        if constexpr (BYTES == 16) {
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "l"(p));
        } else if constexpr (BYTES == 8) {
            asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];"
                         : "=r"(w[0]), "=r"(w[1]) : "l"(p));
        } else {
#pragma unroll
            for (int i = 0; i < VEC; ++i) w[i] = __float_as_uint(to_f(__ldg(p + i)));
        }
    }
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < WORDS; ++i) w[i] = 0u;
    }
    // element i as fp32
    __device__ __forceinline__ float v(int i) const {
        if constexpr (!RAW || sizeof(T) == 4) {
            return __uint_as_float(w[i]);
        } else {
            return (i & 1) ? __uint_as_float(w[i >> 1] & 0xFFFF0000u)
                           : __uint_as_float(w[i >> 1] << 16);
        }
    }
};

// op(A)[r][kb + kk] for the CTA's K range, as fp32
template <typename T>
__device__ __forceinline__ float load_a(const T* A, const SkParams& p, int r, int kk) {
    return to_f(p.ta ? A[int64_t(kk) * p.lda + r] : A[int64_t(r) * p.lda + kk]);
}

// Store one reduced C element (or its split partial).
__device__ __forceinline__ void store_out(const SkParams& p, int z, int split, int r, int j,
                                          float s) {
    if (p.splits > 1) {
        __stcg(p.ws + ((int64_t(split) * p.batch + z) * p.m + r) * p.n + j, s);
    } else {
        float* dst = p.C + int64_t(z) * p.sc + int64_t(r) * p.ldc + j;
        const float x = p.alpha * s;
        *dst = p.beta == 0.0f ? x : fmaf(p.beta, *dst, x);
    }
}

// Split-K finish, called by every CTA after it stored its partials for
// columns [c_lo, c_hi) of batch z: the CTA that arrives last at this column
// block's counter sums every split's partial in split order 0..S-1 (so the
// result does not depend on which CTA finishes last) and writes C.  The
// counter is reset by that CTA, ready for the next launch on this workspace.
__device__ __forceinline__ void finish_splits(const SkParams& p, int z, int c_lo, int c_hi) {
    __shared__ int s_last;
    __threadfence();  // this CTA's partials are visible device-wide ...
    __syncthreads();
    if (threadIdx.x == 0) {  // ... before its arrival is counted
        unsigned* ctr = p.counters + int64_t(z) * gridDim.x + blockIdx.x;
        const unsigned prev = atomicAdd(ctr, 1u);
        s_last = prev == unsigned(p.splits - 1);
        if (s_last) *ctr = 0u;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int ncols = c_hi - c_lo;
    const int64_t plane = int64_t(p.batch) * p.m * p.n;
    if ((p.n & 3) == 0 && (c_lo & 3) == 0 && (ncols & 3) == 0) {
        // float4 groups of columns, every split's load in flight at once
        const int q = ncols >> 2;
        for (int o = threadIdx.x; o < p.m * q; o += THREADS) {
            const int r = o / q, j = c_lo + 4 * (o % q);
            const float* src = p.ws + (int64_t(z) * p.m + r) * p.n + j;
            float4 sum = __ldcg(reinterpret_cast<const float4*>(src));
            int sp = 1;
            for (; sp + 8 <= p.splits; sp += 8) {
                float4 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    v[u] = __ldcg(reinterpret_cast<const float4*>(src + (sp + u) * plane));
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    sum.x += v[u].x; sum.y += v[u].y; sum.z += v[u].z; sum.w += v[u].w;
                }
            }
            for (; sp < p.splits; ++sp) {
                const float4 v = __ldcg(reinterpret_cast<const float4*>(src + sp * plane));
                sum.x += v.x; sum.y += v.y; sum.z += v.z; sum.w += v.w;
            }
            float* dst = p.C + int64_t(z) * p.sc + int64_t(r) * p.ldc + j;
            const float x[4] = {sum.x, sum.y, sum.z, sum.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float y = p.alpha * x[u];
                dst[u] = p.beta == 0.0f ? y : fmaf(p.beta, dst[u], y);
            }
        }
        return;
    }
    for (int o = threadIdx.x; o < p.m * ncols; o += THREADS) {
        const int r = o / ncols, j = c_lo + o % ncols;
        const float* src = p.ws + (int64_t(z) * p.m + r) * p.n + j;
        float sum = __ldcg(src);
        int sp = 1;
        for (; sp + 8 <= p.splits; sp += 8) {  // 8 loads in flight, added in order
            float v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcg(src + (sp + u) * plane);
#pragma unroll
            for (int u = 0; u < 8; ++u) sum += v[u];
        }
        for (; sp < p.splits; ++sp) sum += __ldcg(src + sp * plane);
        float* dst = p.C + int64_t(z) * p.sc + int64_t(r) * p.ldc + j;
        const float x = p.alpha * sum;
        *dst = p.beta == 0.0f ? x : fmaf(p.beta, *dst, x);
    }
}

// ------------------------------------------------------ B normal (k x n)
// CTA: 32*VEC columns x kr rows. sA[kk][MR] (row kk = the m values of A's
// column kb + kk), zero past m and past ke.  Software pipelined: a warp's
// next RPW B rows are in flight while it multiplies the current ones (the
// first batch is issued before A is staged); FFMA2 pairs adjacent columns.
// resident CTAs per SM the register budget is fixed for (latency hiding)
template <int MR>
constexpr int min_ctas() { return MR >= 4 ? 2 : 3; }

template <typename T, int MR, int VEC, int RPW>
__global__ void __launch_bounds__(THREADS, min_ctas<MR>())
skinny_bn_kernel(const SkParams p) {
    extern __shared__ __align__(16) float smem[];
    constexpr int NBLK = 32 * VEC;
    constexpr int STEP = WARPS * RPW;
    constexpr int H = VEC / 2;  // FFMA2 column pairs per thread (VEC even)
    const int z = blockIdx.z, split = blockIdx.y;
    const int n0 = blockIdx.x * NBLK;
    const int kb = split * p.kr;
    const int ke = min(p.k, kb + p.kr);
    const int rows = ke - kb;
    const int rows_pad = (rows + STEP - 1) / STEP * STEP;
    const T* A = static_cast<const T*>(p.A) + int64_t(z) * p.sa;
    const T* B = static_cast<const T*>(p.B) + int64_t(z) * p.sb;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int col = n0 + lane * VEC;
    const bool col_ok = col < p.n;  // n % VEC == 0 whenever VEC > 1
    const T* bcol = B + col + int64_t(kb) * p.ldb;
    auto load_rows = [&](Vec<T, VEC>* b, int k0) {
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
            if (col_ok && k0 + i < rows) b[i].load(bcol + int64_t(k0 + i) * p.ldb);
            else b[i].zero();
        }
    };
    Vec<T, VEC> b[RPW];
    int k0 = warp * RPW;
    load_rows(b, k0);  // in flight while A is staged

    // stage A: index runs along A's contiguous dimension
    for (int i = threadIdx.x; i < rows_pad * MR; i += THREADS) {
        int kk, r;
        if (p.ta) { kk = i / MR; r = i % MR; }   // A stored k x m: m contiguous
        else      { r = i / rows_pad; kk = i % rows_pad; }
        smem[kk * MR + r] = (r < p.m && kk < rows) ? load_a(A, p, r, kb + kk) : 0.0f;
    }
    __syncthreads();

    float acc[MR][VEC];
#pragma unroll
    for (int r = 0; r < MR; ++r)
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[r][v] = 0.0f;

#pragma unroll 2
    for (; k0 < rows_pad; k0 += STEP) {
        Vec<T, VEC> nb[RPW];
        load_rows(nb, k0 + STEP);  // zero-filled past the range
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
            const float* a = smem + (k0 + i) * MR;
#pragma unroll
            for (int r = 0; r < MR; ++r) {
                const float av = a[r];
                if constexpr (VEC % 2 == 0) {
#pragma unroll
                    for (int h = 0; h < H; ++h) {
                        const float2 c = __ffma2_rn(make_float2(av, av),
                                                    make_float2(b[i].v(2 * h), b[i].v(2 * h + 1)),
                                                    make_float2(acc[r][2 * h], acc[r][2 * h + 1]));
                        acc[r][2 * h] = c.x;
                        acc[r][2 * h + 1] = c.y;
                    }
                } else {
#pragma unroll
                    for (int v = 0; v < VEC; ++v) acc[r][v] = fmaf(av, b[i].v(v), acc[r][v]);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < RPW; ++i) b[i] = nb[i];
    }
    __syncthreads();  // A no longer needed: reuse smem for the warp partials

    float* red = smem;  // [WARPS][MR][NBLK]
#pragma unroll
    for (int r = 0; r < MR; ++r)
#pragma unroll
        for (int v = 0; v < VEC; ++v) red[(warp * MR + r) * NBLK + lane * VEC + v] = acc[r][v];
    __syncthreads();
    for (int o = threadIdx.x; o < MR * NBLK; o += THREADS) {
        const int r = o / NBLK, c = o % NBLK;
        if (r >= p.m || n0 + c >= p.n) continue;
        float s = red[r * NBLK + c];
#pragma unroll
        for (int w = 1; w < WARPS; ++w) s += red[(w * MR + r) * NBLK + c];
        store_out(p, z, split, r, n0 + c, s);
    }
    if (p.splits > 1) finish_splits(p, z, n0, min(n0 + NBLK, p.n));
}

// -------------------------------------------------- B transposed (n x k)
// CTA: groups x WARPS*NCW columns x kr rows; sA[r][kk] with row pitch
// rows_pad (fp32).  A warp owns NCW columns per group and its lanes split K;
// the (group, K step) iterations are flattened so the next step's B vectors
// (also the next group's first) are in flight during the current FMAs.
// FFMA2 pairs adjacent k (even / odd partial sums, added once at the end).
template <typename T, int MR, int VEC, int NCW, int UNROLL>
__global__ void __launch_bounds__(THREADS, min_ctas<MR>())
skinny_bt_kernel(const SkParams p) {
    extern __shared__ __align__(16) float smem[];
    constexpr int STEP = 32 * VEC;  // K elements per warp-wide vector step
    constexpr int KSTEP = STEP * UNROLL;
    constexpr int CPG = WARPS * NCW;  // columns per group
    const int z = blockIdx.z, split = blockIdx.y;
    const int kb = split * p.kr;
    const int ke = min(p.k, kb + p.kr);
    const int rows = ke - kb;
    const int rows_pad = (rows + KSTEP - 1) / KSTEP * KSTEP;
    const T* A = static_cast<const T*>(p.A) + int64_t(z) * p.sa;
    const T* B = static_cast<const T*>(p.B) + int64_t(z) * p.sb + kb;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cbase = blockIdx.x * p.groups * CPG;
    const int groups = min(p.groups, (p.n - cbase + CPG - 1) / CPG);
    const int iters = rows_pad / KSTEP;
    const int total = groups * iters;

    auto load_step = [&](Vec<T, VEC> (*b)[NCW], int t) {
        const int grp = t / iters;
        const int k0 = (t - grp * iters) * KSTEP + lane * VEC;
        const int c0 = cbase + grp * CPG + warp * NCW;
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
#pragma unroll
            for (int c = 0; c < NCW; ++c) {
                const int kk = k0 + u * STEP;
                if (t < total && c0 + c < p.n && kk < rows)  // k % VEC == 0 whenever VEC > 1
                    b[u][c].load(B + int64_t(c0 + c) * p.ldb + kk);
                else
                    b[u][c].zero();
            }
    };
    Vec<T, VEC> b[UNROLL][NCW];
    load_step(b, 0);  // in flight while A is staged

    for (int i = threadIdx.x; i < rows_pad * MR; i += THREADS) {
        int kk, r;
        if (p.ta) { kk = i / MR; r = i % MR; }
        else      { r = i / rows_pad; kk = i % rows_pad; }
        smem[r * rows_pad + kk] = (r < p.m && kk < rows) ? load_a(A, p, r, kb + kk) : 0.0f;
    }
    __syncthreads();

    float acc[MR][NCW][2];
#pragma unroll
    for (int r = 0; r < MR; ++r)
#pragma unroll
        for (int c = 0; c < NCW; ++c) acc[r][c][0] = acc[r][c][1] = 0.0f;

    for (int t = 0; t < total; ++t) {
        Vec<T, VEC> nb[UNROLL][NCW];
        load_step(nb, t + 1);
        const int grp = t / iters;
        const int k0 = (t - grp * iters) * KSTEP + lane * VEC;
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const int kk = k0 + u * STEP;
#pragma unroll
            for (int r = 0; r < MR; ++r) {
                float a[VEC];
                if constexpr (VEC == 4) {
                    const float4 q = *reinterpret_cast<const float4*>(smem + r * rows_pad + kk);
                    a[0] = q.x; a[1] = q.y; a[2] = q.z; a[3] = q.w;
                } else {
#pragma unroll
                    for (int v = 0; v < VEC; ++v) a[v] = smem[r * rows_pad + kk + v];
                }
#pragma unroll
                for (int c = 0; c < NCW; ++c) {
                    if constexpr (VEC % 2 == 0) {
#pragma unroll
                        for (int h = 0; h < VEC / 2; ++h) {
                            const float2 s2 = __ffma2_rn(
                                make_float2(a[2 * h], a[2 * h + 1]),
                                make_float2(b[u][c].v(2 * h), b[u][c].v(2 * h + 1)),
                                make_float2(acc[r][c][0], acc[r][c][1]));
                            acc[r][c][0] = s2.x;
                            acc[r][c][1] = s2.y;
                        }
                    } else {
#pragma unroll
                        for (int v = 0; v < VEC; ++v)
                            acc[r][c][0] = fmaf(a[v], b[u][c].v(v), acc[r][c][0]);
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
#pragma unroll
            for (int c = 0; c < NCW; ++c) b[u][c] = nb[u][c];

        if (t - grp * iters == iters - 1) {  // last K step of this group: reduce, store
            const int c0 = cbase + grp * CPG + warp * NCW;
#pragma unroll
            for (int r = 0; r < MR; ++r)
#pragma unroll
                for (int c = 0; c < NCW; ++c) {
                    float v = acc[r][c][0] + acc[r][c][1];
                    // warp-shuffle butterfly over the 32 lanes' K slices
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1)
                        v += __shfl_xor_sync(0xffffffffu, v, off);
                    // lane (r * NCW + c) % 32 stores element (r, c)
                    if (lane == (r * NCW + c) % 32 && r < p.m && c0 + c < p.n)
                        store_out(p, z, split, r, c0 + c, v);
                    acc[r][c][0] = acc[r][c][1] = 0.0f;
                }
        }
    }
    if (p.splits > 1) finish_splits(p, z, cbase, min(cbase + groups * CPG, p.n));
}

// ------------------------------------------------------------------ host
static std::atomic<int> g_mode{1};

int32_t set_mode(int32_t mode) {
    if (mode < 0 || mode > 2) return -1;
    return g_mode.exchange(mode);
}

bool eligible(kp_family fam, const GemmProblem& g) {
    const int mode = g_mode.load(std::memory_order_relaxed);
    if (mode == 0 || g.m > MAX_M) return false;
    if (mode == 2) return true;
    // auto: FC-like shapes -- enough B to stream that the 128-row tiles of
    // the config families would mostly idle.  FP32 SIMT: every m <= 16 (the
    // tile configs stream B at < 1 TB/s there).  TF32 / BF16: m <= 4 only --
    // from m = 8 the SIMT FMAs of the small-M kernels, not HBM, are the
    // limit and the split-K tcgen05 tiles are as fast or faster (measured,
    // profiles/skinny_r02.md).
    const int64_t m_max = fam == KP_F32_SIMT ? MAX_M : 4;
    return g.m <= m_max && g.k >= 64 && g.n >= 64;
}

// Per-device split-K workspace: WS_SLOTS slots, each partials + counters;
// launches take slots round-robin (concurrent split launches on different
// streams never share one unless more than WS_SLOTS are in flight).
constexpr size_t WS_SLOTS = 4;
constexpr size_t WS_SLOT_BYTES = size_t(32) << 20;  // partials
constexpr size_t WS_COUNTERS = 65536;                // column blocks x batch per launch

static kp_status ws_reserve(float** ws, unsigned** counters) {
    static std::mutex mu;
    static char* base[64] = {nullptr};
    static unsigned next[64] = {0};
    const int dev = current_device();
    if (dev < 0 || dev >= 64) return fail(KP_ERR_CUDA, "skinny: bad device");
    constexpr size_t slot = WS_SLOT_BYTES + WS_COUNTERS * sizeof(unsigned);
    std::lock_guard<std::mutex> lock(mu);
    if (!base[dev]) {
        void* ptr = nullptr;
        if (cudaMalloc(&ptr, WS_SLOTS * slot) != cudaSuccess)
            return check_launch("skinny workspace cudaMalloc");
        if (cudaMemset(ptr, 0, WS_SLOTS * slot) != cudaSuccess)
            return check_launch("skinny workspace cudaMemset");
        base[dev] = static_cast<char*>(ptr);
    }
    char* s = base[dev] + (next[dev]++ % WS_SLOTS) * slot;
    *ws = reinterpret_cast<float*>(s);
    *counters = reinterpret_cast<unsigned*>(s + WS_SLOT_BYTES);
    return KP_OK;
}

static kp_status reserve_splits(const GemmProblem& g, int64_t blocks, SkParams& p) {
    if (p.splits == 1) return KP_OK;
    if (size_t(p.splits) * g.batch * g.m * g.n * 4 > WS_SLOT_BYTES || size_t(blocks) > WS_COUNTERS)
        return fail(KP_ERR_UNSUPPORTED, "skinny: split workspace too small");
    return ws_reserve(&p.ws, &p.counters);
}

// Opt every (kernel, device) into > 48 KB of dynamic shared memory once.
template <typename K>
static kp_status set_smem(K kern) {
    static std::mutex mu;
    static std::vector<std::pair<const void*, int>> done;
    const void* key = reinterpret_cast<const void*>(kern);
    const int dev = current_device();
    std::lock_guard<std::mutex> lock(mu);
    for (const auto& e : done)
        if (e.first == key && e.second == dev) return KP_OK;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, MAX_SMEM) != cudaSuccess)
        return check_launch("skinny cudaFuncSetAttribute");
    done.emplace_back(key, dev);
    return KP_OK;
}

// K ranges: one full wave of CTAs (occupancy x SMs) when the column blocks
// alone cannot fill it -- every CTA streams the same number of B rows, so
// the wave ends together -- with each range >= min_rows and its A slice
// within the shared-memory budget (more waves only when K forces it).
template <typename K, typename SmemFn>
static void plan_splits(K kern, const GemmProblem& g, int64_t ctas_per_split, int step,
                        int64_t max_rows, int64_t min_rows, SmemFn smem_for, SkParams& p) {
    const int64_t s_min = std::max<int64_t>(1, (g.k + max_rows - 1) / max_rows);
    const int64_t s_max = std::max<int64_t>(s_min, g.k / min_rows);
    int64_t s = s_min;
    for (int it = 0; it < 2; ++it) {
        int64_t rows = (g.k + s - 1) / s;
        rows = (rows + step - 1) / step * step;
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, THREADS,
                                                          smem_for(rows)) != cudaSuccess || occ < 1)
            occ = 1;
        const int64_t slots = int64_t(occ) * sm_count();
        if (slots / ctas_per_split >= s_min) {
            s = std::min(s_max, slots / ctas_per_split);  // one full wave
        } else {  // K forces more ranges: fill whole waves
            const int64_t waves = (s_min * ctas_per_split + slots - 1) / slots;
            s = std::min(s_max, std::max(s_min, waves * slots / ctas_per_split));
        }
        s = std::min<int64_t>(s, 4096);
    }
    int64_t rows = (g.k + s - 1) / s;
    rows = (rows + step - 1) / step * step;
    p.kr = int(rows);
    p.splits = int((g.k + rows - 1) / rows);
}

template <typename T, int MR, int VEC, int RPW>
static kp_status launch_bn(const GemmProblem& g, SkParams& p, cudaStream_t s) {
    constexpr int NBLK = 32 * VEC;
    constexpr int STEP = WARPS * RPW;
    const int64_t cols = (g.n + NBLK - 1) / NBLK;
    const int64_t red_bytes = int64_t(WARPS) * MR * NBLK * 4;
    const int64_t max_rows = std::max<int64_t>(STEP, (MAX_SMEM / (MR * 4)) / STEP * STEP);
    auto kern = skinny_bn_kernel<T, MR, VEC, RPW>;
    auto smem_for = [&](int64_t rows) {
        const int64_t pad = (rows + STEP - 1) / STEP * STEP;
        return size_t(std::max<int64_t>(pad * MR * 4, red_bytes));
    };
    kp_status st;
    if ((st = set_smem(kern)) != KP_OK) return st;
    plan_splits(kern, g, cols * g.batch, STEP, std::min<int64_t>(max_rows, 8192), 2 * STEP,
                smem_for, p);
    if ((st = reserve_splits(g, cols * g.batch, p)) != KP_OK) return st;
    kern<<<dim3(unsigned(cols), unsigned(p.splits), unsigned(g.batch)), THREADS, smem_for(p.kr), s>>>(p);
    note_launch();
    return check_launch("skinny_bn_kernel");
}

template <typename T, int MR, int VEC, int NCW, int UNROLL>
static kp_status launch_bt(const GemmProblem& g, SkParams& p, cudaStream_t s) {
    constexpr int STEP = 32 * VEC * UNROLL;
    // ~128 columns per CTA share its staged A slice, fewer when the column
    // count alone would not give every SM a CTA
    const int64_t groups_all = (g.n + WARPS * NCW - 1) / (WARPS * NCW);
    const int64_t grp = std::max<int64_t>(1, 128 / (WARPS * NCW));
    p.groups = int(grp);
    const int64_t cols = (groups_all + grp - 1) / grp;
    const int64_t max_rows = std::max<int64_t>(STEP, (MAX_SMEM / (MR * 4)) / STEP * STEP);
    auto kern = skinny_bt_kernel<T, MR, VEC, NCW, UNROLL>;
    auto smem_for = [&](int64_t rows) {
        return size_t((rows + STEP - 1) / STEP * STEP * MR * 4);
    };
    kp_status st;
    if ((st = set_smem(kern)) != KP_OK) return st;
    plan_splits(kern, g, cols * g.batch, STEP, std::min<int64_t>(max_rows, 8192), STEP, smem_for,
                p);
    if ((st = reserve_splits(g, cols * g.batch, p)) != KP_OK) return st;
    kern<<<dim3(unsigned(cols), unsigned(p.splits), unsigned(g.batch)), THREADS, smem_for(p.kr), s>>>(p);
    note_launch();
    return check_launch("skinny_bt_kernel");
}

static bool aligned_to(const void* ptr, int64_t bytes) {
    return (reinterpret_cast<uintptr_t>(ptr) % uintptr_t(bytes)) == 0;
}

template <typename T, int MR>
static kp_status by_layout(const GemmProblem& g, SkParams& p, cudaStream_t s) {
    constexpr int ES = int(sizeof(T));
    // vector width: 16-byte B loads (8-byte for bf16 at MR 16, register budget)
    constexpr int VB = (ES == 2 && MR >= 8) ? 4 : 16 / ES;
    if (!g.tb) {
        const bool vec = g.n % VB == 0 && (g.ldb * ES) % (VB * ES) == 0 &&
                         (g.batch == 1 || (g.sb * ES) % (VB * ES) == 0) && aligned_to(g.B, VB * ES);
        constexpr int RPW = MR >= 16 ? 4 : 8;
        return vec ? launch_bn<T, MR, VB, RPW>(g, p, s) : launch_bn<T, MR, 1, 8>(g, p, s);
    }
    constexpr int VT = 16 / ES;
    const bool vec = g.k % VT == 0 && (g.ldb * ES) % 16 == 0 &&
                     (g.batch == 1 || (g.sb * ES) % 16 == 0) && aligned_to(g.B, 16);
    constexpr int NCW = MR <= 4 ? 4 : 2;
    if (vec) return launch_bt<T, MR, (VT > 4 ? 4 : VT), NCW, 2>(g, p, s);
    return launch_bt<T, MR, 1, NCW, 4>(g, p, s);
}

template <typename T>
static kp_status by_rows(const GemmProblem& g, SkParams& p, cudaStream_t s) {
    if (g.m <= 1) return by_layout<T, 1>(g, p, s);
    if (g.m <= 2) return by_layout<T, 2>(g, p, s);
    if (g.m <= 4) return by_layout<T, 4>(g, p, s);
    if (g.m <= 8) return by_layout<T, 8>(g, p, s);
    return by_layout<T, 16>(g, p, s);
}

kp_status launch(kp_family fam, const GemmProblem& g, cudaStream_t s) {
    if (fam != KP_F32_SIMT && fam != KP_TF32_TC && fam != KP_BF16_TC)
        return fail(KP_ERR_INVALID_ARG, "unknown kernel family");
    if (g.m > MAX_M) return fail(KP_ERR_UNSUPPORTED, "skinny path: m must be <= 16");
    if (g.k > 0x7fffffffLL || g.n > 0x7fffffffLL || g.batch > 65535)
        return fail(KP_ERR_BAD_SHAPE, "skinny path: k, n must fit in int32, batch <= 65535");
    SkParams p;
    p.A = g.A; p.B = g.B; p.C = g.C; p.ws = nullptr; p.counters = nullptr;
    p.m = int(g.m); p.n = int(g.n); p.k = int(g.k);
    p.ta = g.ta ? 1 : 0;
    p.lda = g.lda; p.ldb = g.ldb; p.ldc = g.ldc;
    p.sa = g.sa; p.sb = g.sb; p.sc = g.sc;
    p.alpha = g.alpha; p.beta = g.beta;
    p.batch = int(g.batch);
    p.splits = 1; p.kr = p.k; p.groups = 1;
    return fam == KP_BF16_TC ? by_rows<__nv_bfloat16>(g, p, s) : by_rows<float>(g, p, s);
}

}  // namespace skinny
}  // namespace kp
