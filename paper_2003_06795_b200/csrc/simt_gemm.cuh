// K1: FP32 FFMA register-tiled GEMM family (the paper's 640-point space).
//
// Geometry follows the reference's only executable description of the kernel
// family, synthetic.analytic_perf (reference pkg/src/kernelprune/synthetic.py:
// 65-70):
//   * each thread (work item) owns a row_tile x col_tile block of C,
//   * a work-group of wg_rows x wg_cols threads owns a
//     (row_tile*wg_rows) x (col_tile*wg_cols) block of C,
//   * K is consumed `acc` values per register step.
// row_tile/col_tile/acc are template parameters (64 kernels per operand
// layout); the work-group shape is a runtime launch parameter, as in the paper
// ("can be set at runtime and do not require additional kernels").
//
// B200 mapping:
//   * global -> shared through a 2/3-stage cp.async ring (16-byte copies when
//     rows are 16-byte aligned, 4-byte zero-filling copies otherwise), shared
//     K depth BK = 16 (a multiple of every acc);
//   * shared tiles keep the operand's global layout (no transposes), and each
//     thread's rows/cols are laid out so its fragment reads are vectorised
//     along the operand's contiguous axis and bank-conflict free:
//       A k-contiguous (NN):  rows ty + i*wg_rows, float-vectors of `acc`
//       A m-contiguous (TA):  rows in 4-chunks q*4*wg_rows + ty*4 + e
//                             (ty*row_tile + i when row_tile < 4)
//       B n-contiguous (NN):  cols in 4-chunks q*4*wg_cols + tx*4 + e
//                             (tx*col_tile + j when col_tile < 4)
//       B k-contiguous (TB):  cols tx + j*wg_cols,  float-vectors of `acc`
//   * every C element accumulates its K products in increasing k with fmaf,
//     starting from +0, so results are bit-identical to the sequential-fmaf
//     oracle (oracle/gemm_ref.c); K/M/N tails are zero-filled in shared memory.
#pragma once

#include "kp_internal.cuh"

namespace kp {
namespace simt {

constexpr int BK = 16;      // shared-memory K depth per pipeline stage
constexpr int LOG_BK = 4;
constexpr int PAD = 4;      // floats of padding per shared row (keeps 16 B alignment)
constexpr int GROUP_M = 8;  // tile raster: 8 m-tiles share a sweep over n

struct Params {
    const float* A;
    const float* B;
    float* C;
    int M, N, K;
    int64_t lda, ldb, ldc, sa, sb, sc;
    float alpha, beta;
    int wgr, wgc, log_wgc;
    int log_bm, log_bn;
    int stages;
    int vecA, vecB, vecC;
    int tiles_m, tiles_n;
    int a_stride, b_stride;  // floats per shared row
    int a_elems, b_elems;    // floats per stage
};

// Cooperative copy of a rows x cols block (cols = 1 << log_cols contiguous in
// global memory) into shared memory with row stride s_stride. Elements with
// r >= row_lim or c >= col_lim are written as zero.
__device__ __forceinline__ void load_tile(float* s, int s_stride, const float* g, int64_t g_ld,
                                          int rows, int log_cols, int row_lim, int col_lim,
                                          bool vec, int tid, int nthr) {
    if (vec && log_cols >= 2) {
        const int log_cpr = log_cols - 2;
        const int total = rows << log_cpr;
        for (int idx = tid; idx < total; idx += nthr) {
            const int r = idx >> log_cpr;
            const int c = (idx & ((1 << log_cpr) - 1)) << 2;
            int valid = 0;
            if (r < row_lim) valid = min(max(col_lim - c, 0), 4);
            const float* src = valid ? g + (int64_t)r * g_ld + c : g;
            cp_async16(s + r * s_stride + c, src, valid * 4);
        }
    } else {
        const int cols = 1 << log_cols;
        const int total = rows << log_cols;
        for (int idx = tid; idx < total; idx += nthr) {
            const int r = idx >> log_cols;
            const int c = idx & (cols - 1);
            const bool ok = (r < row_lim) && (c < col_lim);
            const float* src = ok ? g + (int64_t)r * g_ld + c : g;
            cp_async4(s + r * s_stride + c, src, ok ? 4 : 0);
        }
    }
}

// Copy one pipeline stage of an operand tile into shared memory. The tile is
// rows x cols (cols = 1 << log_cols contiguous in global memory, row pitch
// ld); KCOL says whether K runs along the columns (A normal, B transposed) or
// along the rows (A transposed, B normal); `lim` is the in-range extent of the
// non-K axis. Fast path (16-byte copies, >= one thread per 4-float column
// chunk, <= 8 chunks per thread): a thread's chunks share one column position
// and sit dr rows apart, so the per-stage cost is a few integer ops plus the
// cp.async instructions; everything else is block-uniform. Stateless on
// purpose: keeping per-thread copy plans live costs registers the 8x8
// accumulator tiles need (measured: 128 -> 200+ registers).
template <bool KCOL>
__device__ __forceinline__ void copy_stage(float* s, int s_stride, const float* tile, int64_t ld,
                                           int rows, int log_cols, int lim, int k0, int K,
                                           bool vec, int tid, int nthr) {
    const int log_cpr = log_cols - 2;
    if (vec && log_cpr >= 0 && (nthr >> log_cpr) > 0 && (rows << log_cpr) <= 8 * nthr) {
        const int r0 = tid >> log_cpr;
        const int c0 = (tid & ((1 << log_cpr) - 1)) << 2;
        const int dr = nthr >> log_cpr;
        const int total = rows << log_cpr;
        const int n = total >= nthr ? total / nthr : (tid < total ? 1 : 0);
        float* sp = s + r0 * s_stride + c0;
        const int s_step = dr * s_stride;
        const int64_t g_step = (int64_t)dr * ld;
        if constexpr (KCOL) {
            const float* gp = tile + (int64_t)r0 * ld + c0 + k0;
            const int kbytes = min(max(K - k0 - c0, 0), 4) * 4;
            const int rv = lim - r0;  // chunk c in range while c*dr < rv
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                if (c < n) {
                    const int bytes = c * dr < rv ? kbytes : 0;
                    cp_async16(sp + c * s_step, bytes ? gp + c * g_step : tile, bytes);
                }
            }
        } else {
            const float* gp = tile + (int64_t)(r0 + k0) * ld + c0;
            const int cbytes = min(max(lim - c0, 0), 4) * 4;
            const int kv = K - k0 - r0;  // chunk c in range while c*dr < kv
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                if (c < n) {
                    const int bytes = c * dr < kv ? cbytes : 0;
                    cp_async16(sp + c * s_step, bytes ? gp + c * g_step : tile, bytes);
                }
            }
        }
    } else if constexpr (KCOL) {
        load_tile(s, s_stride, tile + k0, ld, rows, log_cols, lim, K - k0, vec, tid, nthr);
    } else {
        load_tile(s, s_stride, tile + (int64_t)k0 * ld, ld, rows, log_cols, K - k0, lim, vec, tid,
                  nthr);
    }
}

// Vector shared-memory load of W consecutive floats (W in 1,2,4,8).
template <int W>
__device__ __forceinline__ void lds(const float* p, float* out) {
    if constexpr (W == 1) {
        out[0] = p[0];
    } else if constexpr (W == 2) {
        const float2 v = *reinterpret_cast<const float2*>(p);
        out[0] = v.x; out[1] = v.y;
    } else {
#pragma unroll
        for (int q = 0; q < W / 4; ++q) {
            const float4 v = reinterpret_cast<const float4*>(p)[q];
            out[4 * q + 0] = v.x; out[4 * q + 1] = v.y;
            out[4 * q + 2] = v.z; out[4 * q + 3] = v.w;
        }
    }
}

// Thread -> output row / column maps (see the header comment): operands read
// along their contiguous axis use 4-wide chunks strided by 4*work-group so a
// quarter-warp's 16-byte shared loads are contiguous (conflict free).
template <bool TA, int RT>
__device__ __forceinline__ int row_of(int i, int ty, int wgr) {
    if constexpr (!TA) return ty + i * wgr;
    else if constexpr (RT >= 4) return (i / 4) * 4 * wgr + ty * 4 + (i % 4);
    else return ty * RT + i;
}
template <bool TB, int CT>
__device__ __forceinline__ int col_of(int j, int tx, int wgc) {
    if constexpr (TB) return tx + j * wgc;
    else if constexpr (CT >= 4) return (j / 4) * 4 * wgc + tx * 4 + (j % 4);
    else return tx * CT + j;
}

__device__ __forceinline__ float epilogue(float acc, float alpha, float beta, const float* c_old) {
    const float v = alpha * acc;
    return beta == 0.0f ? v : fmaf(beta, *c_old, v);
}

template <int ACC, int RT, int CT, bool TA, bool TB>
__global__ void __launch_bounds__(256, 2) simt_gemm_kernel(const Params p) {
    extern __shared__ __align__(16) float smem[];
    const int tid = threadIdx.x;
    const int nthr = p.wgr * p.wgc;
    const int ty = tid >> p.log_wgc;
    const int tx = tid & (p.wgc - 1);

    // grouped raster over (tiles_m x tiles_n) for L2 reuse of A rows / B cols
    const int tile = blockIdx.x;
    const int per_group = GROUP_M * p.tiles_n;
    const int group = tile / per_group;
    const int first_m = group * GROUP_M;
    const int gsz = min(p.tiles_m - first_m, GROUP_M);
    const int in_group = tile - group * per_group;
    const int tm = first_m + in_group % gsz;
    const int tn = in_group / gsz;

    const int BM = RT * p.wgr;
    const int BN = CT * p.wgc;
    const int m0 = tm * BM;
    const int n0 = tn * BN;
    const int64_t bz = blockIdx.z;
    const float* __restrict__ A = p.A + bz * p.sa;
    const float* __restrict__ B = p.B + bz * p.sb;
    float* __restrict__ C = p.C + bz * p.sc;

    float* sA = smem;
    float* sB = smem + p.stages * p.a_elems;
    const int KT = (p.K + BK - 1) >> LOG_BK;

    // A: k-contiguous rows of m (normal) or m-contiguous rows of k (TA);
    // B: n-contiguous rows of k (normal) or k-contiguous rows of n (TB).
    auto issue = [&](int kt, int stage) {
        const int k0 = kt << LOG_BK;
        float* a_dst = sA + stage * p.a_elems;
        float* b_dst = sB + stage * p.b_elems;
        if constexpr (!TA)
            copy_stage<true>(a_dst, p.a_stride, A + (int64_t)m0 * p.lda, p.lda, BM, LOG_BK,
                             p.M - m0, k0, p.K, p.vecA, tid, nthr);
        else
            copy_stage<false>(a_dst, p.a_stride, A + m0, p.lda, BK, p.log_bm, p.M - m0, k0, p.K,
                              p.vecA, tid, nthr);
        if constexpr (!TB)
            copy_stage<false>(b_dst, p.b_stride, B + n0, p.ldb, BK, p.log_bn, p.N - n0, k0, p.K,
                              p.vecB, tid, nthr);
        else
            copy_stage<true>(b_dst, p.b_stride, B + (int64_t)n0 * p.ldb, p.ldb, BN, LOG_BK,
                             p.N - n0, k0, p.K, p.vecB, tid, nthr);
    };

    float acc[RT][CT];
#pragma unroll
    for (int i = 0; i < RT; ++i)
#pragma unroll
        for (int j = 0; j < CT; ++j) acc[i][j] = 0.0f;

    const int S = p.stages;
    for (int s = 0; s < S - 1; ++s) {
        if (s < KT) issue(s, s);
        cp_async_commit();
    }

    int rd = 0, wr = S - 1;  // stage being read / written
    for (int kt = 0; kt < KT; ++kt) {
        if (S == 3) cp_async_wait<1>(); else cp_async_wait<0>();
        __syncthreads();
        if (kt + S - 1 < KT) issue(kt + S - 1, wr);
        cp_async_commit();
        wr = (wr + 1 == S) ? 0 : wr + 1;
        const float* a_s = sA + rd * p.a_elems;
        const float* b_s = sB + rd * p.b_elems;
        rd = (rd + 1 == S) ? 0 : rd + 1;
#pragma unroll
        for (int kb = 0; kb < BK; kb += ACC) {
            float a[RT][ACC];
            float b[ACC][CT];
            if constexpr (!TA) {
#pragma unroll
                for (int i = 0; i < RT; ++i)
                    lds<ACC>(a_s + (ty + i * p.wgr) * p.a_stride + kb, a[i]);
            } else {
#pragma unroll
                for (int kk = 0; kk < ACC; ++kk) {
                    float t[RT];
                    if constexpr (RT >= 4) {
#pragma unroll
                        for (int q = 0; q < RT / 4; ++q)
                            lds<4>(a_s + (kb + kk) * p.a_stride + q * 4 * p.wgr + ty * 4, t + 4 * q);
                    } else {
                        lds<RT>(a_s + (kb + kk) * p.a_stride + ty * RT, t);
                    }
#pragma unroll
                    for (int i = 0; i < RT; ++i) a[i][kk] = t[i];
                }
            }
            if constexpr (!TB) {
#pragma unroll
                for (int kk = 0; kk < ACC; ++kk) {
                    if constexpr (CT >= 4) {
#pragma unroll
                        for (int q = 0; q < CT / 4; ++q)
                            lds<4>(b_s + (kb + kk) * p.b_stride + q * 4 * p.wgc + tx * 4, b[kk] + 4 * q);
                    } else {
                        lds<CT>(b_s + (kb + kk) * p.b_stride + tx * CT, b[kk]);
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < CT; ++j) {
                    float t[ACC];
                    lds<ACC>(b_s + (tx + j * p.wgc) * p.b_stride + kb, t);
#pragma unroll
                    for (int kk = 0; kk < ACC; ++kk) b[kk][j] = t[kk];
                }
            }
#pragma unroll
            for (int kk = 0; kk < ACC; ++kk)
#pragma unroll
                for (int i = 0; i < RT; ++i)
#pragma unroll
                    for (int j = 0; j < CT; ++j) acc[i][j] = fmaf(a[i][kk], b[kk][j], acc[i][j]);
        }
    }
    cp_async_wait<0>();

    // epilogue: C = alpha*acc (+ beta*C)
#pragma unroll
    for (int i = 0; i < RT; ++i) {
        const int m = m0 + row_of<TA, RT>(i, ty, p.wgr);
        if (m >= p.M) continue;
        float* crow = C + (int64_t)m * p.ldc;
        if constexpr (!TB && CT >= 4) {
#pragma unroll
            for (int q = 0; q < CT / 4; ++q) {
                const int n = n0 + q * 4 * p.wgc + tx * 4;
                if (p.vecC && n + 3 < p.N) {
                    float4 v;
                    if (p.beta == 0.0f) {
                        v = make_float4(p.alpha * acc[i][4 * q], p.alpha * acc[i][4 * q + 1],
                                        p.alpha * acc[i][4 * q + 2], p.alpha * acc[i][4 * q + 3]);
                    } else {
                        const float4 o = *reinterpret_cast<const float4*>(crow + n);
                        v = make_float4(fmaf(p.beta, o.x, p.alpha * acc[i][4 * q]),
                                        fmaf(p.beta, o.y, p.alpha * acc[i][4 * q + 1]),
                                        fmaf(p.beta, o.z, p.alpha * acc[i][4 * q + 2]),
                                        fmaf(p.beta, o.w, p.alpha * acc[i][4 * q + 3]));
                    }
                    *reinterpret_cast<float4*>(crow + n) = v;
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (n + e < p.N)
                            crow[n + e] = epilogue(acc[i][4 * q + e], p.alpha, p.beta, crow + n + e);
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < CT; ++j) {
                const int n = n0 + col_of<TB, CT>(j, tx, p.wgc);
                if (n < p.N) crow[n] = epilogue(acc[i][j], p.alpha, p.beta, crow + n);
            }
        }
    }
}

inline int ilog2(int v) {
    int l = 0;
    while ((1 << l) < v) ++l;
    return l;
}
inline int round4(int v) { return (v + 3) & ~3; }

// Shared-memory plan for one (layout, tile) combination; used by the
// launcher and by tests through kp_simt_smem_bytes().
struct SmemPlan {
    int a_stride, b_stride, a_elems, b_elems, stages;
    size_t bytes;
};

inline SmemPlan plan_smem(bool ta, bool tb, int bm, int bn) {
    SmemPlan s;
    if (!ta) { s.a_stride = BK + PAD; s.a_elems = bm * s.a_stride; }
    else     { s.a_stride = round4(bm) + PAD; s.a_elems = BK * s.a_stride; }
    if (!tb) { s.b_stride = round4(bn) + PAD; s.b_elems = BK * s.b_stride; }
    else     { s.b_stride = BK + PAD; s.b_elems = bn * s.b_stride; }
    const size_t stage = 4u * size_t(s.a_elems + s.b_elems);
    s.stages = (3 * stage <= 112 * 1024) ? 3 : 2;
    s.bytes = s.stages * stage;
    return s;
}

template <int ACC, int RT, int CT, bool TA, bool TB>
kp_status launch(const GemmProblem& g, int wgr, int wgc, cudaStream_t stream) {
    const int bm = RT * wgr, bn = CT * wgc;
    const SmemPlan sp = plan_smem(TA, TB, bm, bn);
    if (sp.bytes > 227 * 1024) return fail(KP_ERR_UNSUPPORTED, "simt: shared-memory plan too large");
    auto kern = simt_gemm_kernel<ACC, RT, CT, TA, TB>;
    static bool attr_done = false;  // benign race: idempotent attribute set
    if (!attr_done) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess)
            return check_launch("cudaFuncSetAttribute");
        attr_done = true;
    }
    Params p;
    p.A = static_cast<const float*>(g.A);
    p.B = static_cast<const float*>(g.B);
    p.C = g.C;
    p.M = int(g.m); p.N = int(g.n); p.K = int(g.k);
    p.lda = g.lda; p.ldb = g.ldb; p.ldc = g.ldc;
    p.sa = g.sa; p.sb = g.sb; p.sc = g.sc;
    p.alpha = g.alpha; p.beta = g.beta;
    p.wgr = wgr; p.wgc = wgc; p.log_wgc = ilog2(wgc);
    p.log_bm = ilog2(bm); p.log_bn = ilog2(bn);
    p.stages = sp.stages;
    const bool multi = g.batch > 1;
    p.vecA = aligned16(g.A) && g.lda % 4 == 0 && (!multi || g.sa % 4 == 0) && (!TA || bm % 4 == 0);
    p.vecB = aligned16(g.B) && g.ldb % 4 == 0 && (!multi || g.sb % 4 == 0) && (TB || bn % 4 == 0);
    p.vecC = aligned16(g.C) && g.ldc % 4 == 0 && (!multi || g.sc % 4 == 0);
    p.tiles_m = int((g.m + bm - 1) / bm);
    p.tiles_n = int((g.n + bn - 1) / bn);
    p.a_stride = sp.a_stride; p.b_stride = sp.b_stride;
    p.a_elems = sp.a_elems; p.b_elems = sp.b_elems;
    const int64_t tiles = int64_t(p.tiles_m) * p.tiles_n;
    if (tiles > 0x7fffffffLL || g.batch > 65535)
        return fail(KP_ERR_BAD_SHAPE, "simt: grid too large for this work-group tile");
    dim3 grid(unsigned(tiles), 1, unsigned(g.batch));
    kern<<<grid, wgr * wgc, sp.bytes, stream>>>(p);
    note_launch();
    return check_launch("simt_gemm_kernel");
}

}  // namespace simt
}  // namespace kp
