/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the K1 FP32 GEMM family.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library; the product path (libkp.so) never does.
 *
 * What it restates: the matmul the paper's kernel family computes
 * ("each work item computes a tile of the output,
 * accumulating a given number of values in each step"), with the row-major
 * shapes of the reference's ProblemSize (pkg/src/kernelprune/dataset.py:89-100:
 * C is m x n, k is the reduction) and its FLOP convention 2*m*n*k
 * (synthetic.py:110-113).  The GEMM arithmetic itself lives in the
 * un-vendored SYCL-DNN (no pinned version), so GEMM parity
 * is anchored here: every C element accumulates its products in increasing
 * k with a correctly-rounded fmaf, starting from +0.0f; the epilogue is
 *     v = alpha * acc;  if (beta != 0) v = fmaf(beta, c_old, v);
 * which is exactly the order the K1 kernels use, so K1 must match this
 * oracle bit for bit (value equality) for every config and shape.
 *
 * The tcgen05 TF32/BF16 families are checked against the numpy float64
 * oracle (oracle/gemm_oracle.py) within a K-scaled tolerance instead.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* element accessors for the four operand layouts (see include/kp_abi.h) */
static inline float opa(const float* a, int ta, int64_t lda, int64_t i, int64_t p) {
    return ta ? a[p * lda + i] : a[i * lda + p];
}

/* Blocking (AVX2, 4 x 16 register tile): op(A) rows are packed in chunks of
 * MC rows (one OpenMP task each) as k x 4 micro-panels, op(B) as k x 16
 * column panels (zero padded past n; padded columns are never stored).  The
 * micro-kernel keeps the 4 x 16 accumulators in registers for the whole k
 * loop and updates them with _mm256_fmadd_ps -- one correctly rounded fused
 * multiply-add per element and step, i.e. exactly fmaf -- in p = 0, 1, ...,
 * k-1 order starting from +0.0f.  Blocking changes only which independent
 * per-element chains run side by side, never the order inside a chain, so
 * the result is identical to the plain triple loop (pinned by
 * tests/test_oracle.py against exact Python evaluation). */
#include <immintrin.h>

enum { MR = 4, NR = 16, MC = 64 };

static void pack_a(const float* a, int ta, int64_t lda, int64_t i0, int64_t rows, int64_t k,
                   float* dst) {
    for (int64_t r0 = 0; r0 < MC; r0 += MR)
        for (int64_t p = 0; p < k; ++p)
            for (int64_t r = 0; r < MR; ++r) {
                const int64_t i = r0 + r;
                dst[(r0 / MR) * k * MR + p * MR + r] = i < rows ? opa(a, ta, lda, i0 + i, p) : 0.0f;
            }
}

static void pack_b(const float* b, int tb, int64_t ldb, int64_t j0, int64_t cols, int64_t k,
                   float* dst) {
    for (int64_t p = 0; p < k; ++p)
        for (int64_t j = 0; j < NR; ++j)
            dst[p * NR + j] = j < cols ? (tb ? b[(j0 + j) * ldb + p] : b[p * ldb + j0 + j]) : 0.0f;
}

static void micro_4x16(const float* ap, const float* bp, int64_t k, float out[MR][NR]) {
    __m256 c00 = _mm256_setzero_ps(), c01 = _mm256_setzero_ps();
    __m256 c10 = _mm256_setzero_ps(), c11 = _mm256_setzero_ps();
    __m256 c20 = _mm256_setzero_ps(), c21 = _mm256_setzero_ps();
    __m256 c30 = _mm256_setzero_ps(), c31 = _mm256_setzero_ps();
    for (int64_t p = 0; p < k; ++p) {
        const __m256 b0 = _mm256_loadu_ps(bp + p * NR);
        const __m256 b1 = _mm256_loadu_ps(bp + p * NR + 8);
        __m256 av = _mm256_broadcast_ss(ap + p * MR + 0);
        c00 = _mm256_fmadd_ps(av, b0, c00);
        c01 = _mm256_fmadd_ps(av, b1, c01);
        av = _mm256_broadcast_ss(ap + p * MR + 1);
        c10 = _mm256_fmadd_ps(av, b0, c10);
        c11 = _mm256_fmadd_ps(av, b1, c11);
        av = _mm256_broadcast_ss(ap + p * MR + 2);
        c20 = _mm256_fmadd_ps(av, b0, c20);
        c21 = _mm256_fmadd_ps(av, b1, c21);
        av = _mm256_broadcast_ss(ap + p * MR + 3);
        c30 = _mm256_fmadd_ps(av, b0, c30);
        c31 = _mm256_fmadd_ps(av, b1, c31);
    }
    _mm256_storeu_ps(out[0], c00); _mm256_storeu_ps(out[0] + 8, c01);
    _mm256_storeu_ps(out[1], c10); _mm256_storeu_ps(out[1] + 8, c11);
    _mm256_storeu_ps(out[2], c20); _mm256_storeu_ps(out[2] + 8, c21);
    _mm256_storeu_ps(out[3], c30); _mm256_storeu_ps(out[3] + 8, c31);
}

int kp_oracle_gemm_f32(int64_t batch, int64_t m, int64_t k, int64_t n, int32_t ta, int32_t tb,
                       int64_t lda, int64_t ldb, int64_t ldc, int64_t sa, int64_t sb, int64_t sc,
                       float alpha, float beta, const float* A, const float* B, float* C) {
    if (batch < 1 || m < 1 || k < 1 || n < 1) return 2;
    const int64_t chunks = (m + MC - 1) / MC;
    for (int64_t b = 0; b < batch; ++b) {
        const float* a = A + b * sa;
        const float* bb = B + b * sb;
        float* c = C + b * sc;
        int failed = 0;
#pragma omp parallel for schedule(dynamic, 1)
        for (int64_t ch = 0; ch < chunks; ++ch) {
            const int64_t i0 = ch * MC;
            const int64_t rows = (m - i0) < MC ? (m - i0) : MC;
            float* apack = (float*)malloc(sizeof(float) * (size_t)(MC * k));
            float* bpack = (float*)malloc(sizeof(float) * (size_t)(NR * k));
            if (!apack || !bpack) {
                free(apack);
                free(bpack);
#pragma omp atomic write
                failed = 1;
                continue;
            }
            pack_a(a, ta, lda, i0, rows, k, apack);
            for (int64_t j0 = 0; j0 < n; j0 += NR) {
                const int64_t cols = (n - j0) < NR ? (n - j0) : NR;
                pack_b(bb, tb, ldb, j0, cols, k, bpack);
                for (int64_t r0 = 0; r0 < rows; r0 += MR) {
                    float acc[MR][NR];
                    micro_4x16(apack + (r0 / MR) * k * MR, bpack, k, acc);
                    for (int64_t r = 0; r < MR && r0 + r < rows; ++r) {
                        float* crow = c + (i0 + r0 + r) * ldc + j0;
                        for (int64_t j = 0; j < cols; ++j) {
                            float v = alpha * acc[r][j];
                            if (beta != 0.0f) v = fmaf(beta, crow[j], v);
                            crow[j] = v;
                        }
                    }
                }
            }
            free(apack);
            free(bpack);
        }
        if (failed) return 3;
    }
    return 0;
}

/* host threads the oracle uses (bench.py times it on 1 core and on all cores);
 * returns the previous count */
int kp_oracle_set_threads(int n) {
#ifdef _OPENMP
    const int prev = omp_get_max_threads();
    if (n > 0) omp_set_num_threads(n);
    return prev;
#else
    (void)n;
    return 1;
#endif
}
