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

/* element accessors for the four operand layouts (see include/kp_abi.h) */
static inline float opa(const float* a, int ta, int64_t lda, int64_t i, int64_t p) {
    return ta ? a[p * lda + i] : a[i * lda + p];
}

int kp_oracle_gemm_f32(int64_t batch, int64_t m, int64_t k, int64_t n, int32_t ta, int32_t tb,
                       int64_t lda, int64_t ldb, int64_t ldc, int64_t sa, int64_t sb, int64_t sc,
                       float alpha, float beta, const float* A, const float* B, float* C) {
    if (batch < 1 || m < 1 || k < 1 || n < 1) return 2;
    for (int64_t b = 0; b < batch; ++b) {
        const float* a = A + b * sa;
        const float* bb = B + b * sb;
        float* c = C + b * sc;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < m; ++i) {
            float* acc = (float*)calloc((size_t)n, sizeof(float)); /* +0.0f */
            for (int64_t p = 0; p < k; ++p) {
                const float av = opa(a, ta, lda, i, p);
                if (!tb) {
                    const float* brow = bb + p * ldb;
                    for (int64_t j = 0; j < n; ++j) acc[j] = fmaf(av, brow[j], acc[j]);
                } else {
                    for (int64_t j = 0; j < n; ++j) acc[j] = fmaf(av, bb[j * ldb + p], acc[j]);
                }
            }
            float* crow = c + i * ldc;
            for (int64_t j = 0; j < n; ++j) {
                float v = alpha * acc[j];
                if (beta != 0.0f) v = fmaf(beta, crow[j], v);
                crow[j] = v;
            }
            free(acc);
        }
    }
    return 0;
}
