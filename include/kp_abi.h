/*
 * kp_abi.h -- C-ABI of the B200 kernel library (libkp.so).
 *
 * This is the drop-in boundary between the reference's Python host API
 * (kernelprune: dataset / pruning / selector / codegen, reference
 * pkg/src/kernelprune/) and the sm_100a kernels.  Plain C: no CUDA or torch
 * types appear in any signature; device pointers are `void*`/`float*`, the
 * CUDA stream is an opaque `void*` (a cudaStream_t, NULL = legacy default).
 *
 * Reference interfaces replaced (file:line under /root/reference):
 *   kp_config                 <- KernelConfig, pkg/src/kernelprune/dataset.py:63-86
 *                                (field order == canonical order), and the
 *                                generated `<sym>_config` struct, codegen.py:138-144
 *   kp_num_configs/config_at  <- all_configs(), dataset.py:119-126 (640 configs,
 *                                canonical lexicographic order)
 *   kp_config_valid           <- KernelConfig.__post_init__, dataset.py:77-83
 *                                (InvalidConfigValue -> KP_ERR_INVALID_CONFIG)
 *   kp_gemm                   <- the paper's "matmul kernel with a tile config"
 *                                (PAPER.md:116-125); geometry as pinned by
 *                                synthetic.analytic_perf, synthetic.py:65-70
 *   kp_gemm_time              <- per-cell "run config on problem -> runtime_ns",
 *                                the measured twin of synthetic.generate,
 *                                synthetic.py:92-114 (runtime_ns = 2mnk/gflops)
 *   kp_sweep_problem          <- the inner loop of generate() over all configs
 *                                of one problem, synthetic.py:106-113
 *   kp_select / kp_gemm_auto  <- generated `select_kernel(m,k,n)`,
 *                                codegen.py:128-171, compiled into the library
 *                                exactly as harness/parity_main.cpp:21-32,96 does
 *   kp_gemm_skinny            <- no reference counterpart: small-M (FC layer)
 *                                path behind kp_gemm_auto
 *   kp_status                 <- errors.py:4-9 DataError taxonomy; NonPositiveValue
 *                                (dataset.py:95-97) -> KP_ERR_BAD_SHAPE
 *
 * Conventions: every entry point returns a status and never aborts; the
 * library allocates no device memory per call except the stream-ordered
 * staging copy of an unaligned tcgen05 operand (TMEM is allocated/freed inside
 * the tcgen05 kernels; a 256 KB ring of stream-K hand-off flags and a 256 MB
 * tcgen05 split-K workspace are allocated once per device on first use); calls are stream-ordered and reentrant; the message of
 * the last failure on the calling thread is available from kp_last_error().
 */
#ifndef KP_ABI_H
#define KP_ABI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KP_ABI_VERSION 1

/* Same layout as KernelConfig / the generated select_kernel_config struct. */
typedef struct {
    uint32_t acc;       /* K step per register fragment: 1,2,4,8          */
    uint32_t row_tile;  /* output rows per thread: 1,2,4,8                */
    uint32_t col_tile;  /* output cols per thread: 1,2,4,8                */
    uint32_t wg_rows;   /* work-group shape (runtime launch parameter)    */
    uint32_t wg_cols;
} kp_config;

typedef enum {
    KP_F32_SIMT = 0,  /* fp32 in, FFMA register-tiled, fp32 out          */
    KP_TF32_TC  = 1,  /* fp32 in (rounded to tf32), tcgen05 kind::tf32   */
    KP_BF16_TC  = 2   /* bf16 in, tcgen05 kind::f16, fp32 accumulate/out */
} kp_family;

typedef enum {
    KP_OK = 0,
    KP_ERR_INVALID_CONFIG = 1,  /* config outside the family's domain      */
    KP_ERR_BAD_SHAPE = 2,       /* m,k,n,batch < 1 or ld too small          */
    KP_ERR_ALIGNMENT = 3,       /* pointer/ld alignment the family requires */
    KP_ERR_UNSUPPORTED = 4,     /* family/variant not built or no device    */
    KP_ERR_CUDA = 5,            /* a CUDA runtime call failed               */
    KP_ERR_INVALID_ARG = 6      /* null pointer, bad counts                 */
} kp_status;

/*
 * One (optionally strided-batched) GEMM, row-major like numpy:
 *   C[b] = alpha * op(A[b]) @ op(B[b]) + beta * C[b],   b in [0, batch)
 * op(A) is m x k: trans_a == 0 -> A[b][i*lda + p], else A[b][p*lda + i].
 * op(B) is k x n: trans_b == 0 -> B[b][p*ldb + j], else B[b][j*ldb + p].
 * C is m x n: C[b][i*ldc + j].  Strides are in elements.  beta == 0 means C
 * is write-only (never read).
 */
typedef struct {
    int64_t batch, m, k, n;
    int32_t trans_a, trans_b;
    int64_t lda, ldb, ldc;
    int64_t stride_a, stride_b, stride_c;
    float alpha, beta;
} kp_gemm_desc;

/* ---- config space (canonical order = KernelConfig sort order) -------- */
int32_t   kp_abi_version(void);
int32_t   kp_num_configs(kp_family family);
kp_status kp_config_at(kp_family family, int32_t index, kp_config* out);
kp_status kp_config_valid(kp_family family, kp_config cfg);

/* ---- compute ----------------------------------------------------------- */
/* The tcgen05 families load operands with TMA (16-byte aligned base, row and
 * batch pitches).  An operand without that alignment is copied into a
 * stream-ordered temporary (cudaMallocAsync / cudaFreeAsync on `stream`) with
 * zero-padded 16-byte rows first; the result is the same GEMM. */
kp_status kp_gemm(kp_family family, kp_config cfg, const kp_gemm_desc* desc,
                  const void* A, const void* B, float* C, void* stream);

/* Timing loop (K4).  One timed launch that sizes the samples (it also
 * absorbs first-launch costs), `warmup`-1 more untimed launches, then `reps`
 * samples of back-to-back launches (each sample >= min_sample_ns of device time);
 * *runtime_ns = median per-launch device time (CUDA events on `stream`).
 * Cell budget: when reps * (one launch) exceeds max_cell_ns (> 0), the extra
 * warm-ups are skipped and reps shrinks to fit (at least 1 sample), so
 * hopeless configs on big problems cost ~2 launches.  Synchronises `stream`. */
kp_status kp_gemm_time(kp_family family, kp_config cfg, const kp_gemm_desc* desc,
                       const void* A, const void* B, float* C,
                       int32_t warmup, int32_t reps, double min_sample_ns,
                       double max_cell_ns, double* runtime_ns, void* stream);

/* Time every config in `cfgs` on one problem (buffers allocated once by the
 * caller); runtime_ns[i] per config, same timing method as kp_gemm_time,
 * except that a config whose first launch takes over 1 ms and over 8x the
 * best median of this problem so far keeps that single timing. */
kp_status kp_sweep_problem(kp_family family, const kp_config* cfgs, int32_t n_cfgs,
                           const kp_gemm_desc* desc, const void* A, const void* B,
                           float* C, int32_t warmup, int32_t reps,
                           double min_sample_ns, double max_cell_ns,
                           double* runtime_ns, void* stream);

/* kp_sweep_problem with explicit policy flags.  KP_SWEEP_EARLY_EXIT enables
 * the hopeless-config early exit described above (kp_sweep_problem always
 * sets it); without it every config gets the full warm-up + reps statistic --
 * what a sweep split into config ranges needs, since only a call that sees a
 * whole problem knows its best median. */
#define KP_SWEEP_EARLY_EXIT 1
kp_status kp_sweep_problem_ex(kp_family family, const kp_config* cfgs, int32_t n_cfgs,
                              const kp_gemm_desc* desc, const void* A, const void* B,
                              float* C, int32_t warmup, int32_t reps,
                              double min_sample_ns, double max_cell_ns, int32_t flags,
                              double* runtime_ns, void* stream);

/* K1 (FP32 SIMT) tile scheduling.  0 = one output tile per CTA; 1 (default)
 * = ordered stream-K when whole tiles would leave part of the last wave idle:
 * one persistent wave shares the (tile, k-slice) units evenly, a tile split
 * between two CTAs is handed off through C with its k order preserved, so
 * results stay bit-identical to mode 0 (beta == 0 problems only); 2 = ordered
 * stream-K whenever a problem has two or more tiles (tests).  Process-wide;
 * returns the previous mode, or -1 for an unknown mode (left unchanged). */
int32_t   kp_set_schedule(int32_t mode);

/* K2/K3 (tcgen05, 1-CTA configs) split-K.  0 = never; 1 (default) = auto:
 * grids of output tiles filling under half the SMs cut each tile's K range
 * into S contiguous ranges (one CTA each, >= 4 K stages per range, one wave
 * of units), partial tiles go to a per-device workspace and a second kernel
 * sums them in split order 0..S-1 (deterministic); n in
 * [2, 64] = force n splits (clamped to the K stages; tests).  Process-wide;
 * returns the previous mode, or -1 for an invalid mode (left unchanged).
 * Replaces nothing in the reference (its GEMM is external):
 * a scheduling policy inside the kernel family, not a config field. */
int32_t   kp_set_tc_split(int32_t mode);

/* ---- small-M path (m <= 16: fully connected layers at batch 1-16) ----- */
/* A B-streaming kernel pair for any family (fp32 inputs for KP_F32_SIMT and
 * KP_TF32_TC, bf16 for KP_BF16_TC; fp32 FMA accumulate): CTAs own a column
 * block and a K range, stage op(A)'s m rows in shared memory and read B once
 * with 16-byte loads; partial sums meet in a fixed order (warp order through
 * shared memory for B normal, a warp-shuffle butterfly for B transposed,
 * split order through a per-device workspace across K ranges), so results
 * are deterministic but not in the sequential-fmaf order of K1.
 * KP_ERR_UNSUPPORTED when m > 16.  kp_gemm / kp_gemm_time accept the
 * all-zero config KP_SKINNY_CONFIG for the same path (timing, sweeps);
 * kp_config_valid still rejects it (it is not a KernelConfig).
 * Replaces nothing in the reference (its GEMM is external,
 * PAPER.md:112-114): the FC-layer case of the paper's dataset
 * that the tile configs cannot stream at HBM speed. */
#define KP_SKINNY_CONFIG_INIT {0u, 0u, 0u, 0u, 0u}
kp_status kp_gemm_skinny(kp_family family, const kp_gemm_desc* desc, const void* A,
                         const void* B, float* C, void* stream);
/* Whether kp_gemm_auto routes m <= 16 problems to the small-M path:
 * 0 = never, 1 (default) = when k >= 64, n >= 64 and m <= 16 (KP_F32_SIMT)
 * or m <= 4 (KP_TF32_TC / KP_BF16_TC), 2 = every m <= 16 problem.  kp_gemm_auto reports the all-zero config in `chosen`
 * when it took this path.  Returns the previous mode, or -1 (unchanged). */
int32_t   kp_set_skinny(int32_t mode);

/* ---- runtime selection (generated decision-tree header) --------------- */
/* Config the compiled selector picks for (m,k,n); KP_ERR_UNSUPPORTED when no
 * selector is compiled in for this family / transpose variant. */
kp_status kp_select(kp_family family, int32_t trans_a, int32_t trans_b,
                    int64_t m, int64_t k, int64_t n, kp_config* out);
/* kp_select for a strided-batched problem: batch 1 uses the plain selector;
 * batch > 1 the selector trained on the strided-batched dataset whose batch
 * count is closest (log scale) -- one selector per (family, trans, batch)
 * variant, SURVEY H5 -- else the plain one.  kp_gemm_auto calls this with
 * desc->batch. */
kp_status kp_select_ex(kp_family family, int32_t trans_a, int32_t trans_b, int64_t batch,
                       int64_t m, int64_t k, int64_t n, kp_config* out);
/* What kp_gemm_auto launches for this shape: kp_select's config, or the
 * all-zero config when the small-M path takes the problem. */
kp_status kp_auto_config(kp_family family, int32_t trans_a, int32_t trans_b, int64_t batch,
                         int64_t m, int64_t k, int64_t n, kp_config* out);
kp_status kp_gemm_auto(kp_family family, const kp_gemm_desc* desc,
                       const void* A, const void* B, float* C, void* stream,
                       kp_config* chosen /* may be NULL */);

/* ---- im2col front-end (network layers as the selectors' GEMMs) -------- */
/* NCHW input, weights [c_out, c_in*kh*kw] row-major, output NHWC
 * [batch*ho*wo, c_out]; the GEMM is the NT variant (kp_gemm_auto with
 * trans_b = 1), so conv layers run through the compiled NT selector.
 * Tensor-core families: the im2col rows get a 16-byte K pitch (zero
 * columns past K) and unaligned weights are staged (see kp_gemm). */
typedef struct {
    int64_t batch, c_in, h, w, c_out, kh, kw, stride_h, stride_w, pad_h, pad_w;
} kp_conv_desc;
kp_status kp_conv_output_shape(const kp_conv_desc* d, int64_t* ho, int64_t* wo);
/* cols[batch*ho*wo, c_in*kh*kw] (fp32, bf16 for KP_BF16_TC), zero padding. */
kp_status kp_im2col(kp_family family, const kp_conv_desc* d, const void* x, void* cols,
                    void* stream);
/* Same gather with row pitch ldk >= c_in*kh*kw; columns [c_in*kh*kw, ldk)
 * are written as zeros. */
kp_status kp_im2col_pitched(kp_family family, const kp_conv_desc* d, const void* x, void* cols,
                            int64_t ldk, void* stream);
/* Elements of the `cols` workspace kp_conv2d_auto needs: batch*ho*wo rows of
 * c_in*kh*kw, the pitch rounded up to 16 bytes for the tcgen05 families. */
kp_status kp_conv_workspace_elems(kp_family family, const kp_conv_desc* d, int64_t* elems);
kp_status kp_conv2d_auto(kp_family family, const kp_conv_desc* d, const void* x,
                         const void* w, float* y, void* cols /* workspace */, void* stream,
                         kp_config* chosen /* may be NULL */);

/* ---- diagnostics -------------------------------------------------------- */
const char* kp_status_string(kp_status status);
const char* kp_last_error(void);               /* thread-local */
/* Number of kernel launches this process issued through the library. */
int64_t     kp_launch_count(void);
/* Device facts for the sweep sidecar: SM count, max SM clock (kHz),
 * compute capability (major*10+minor). */
kp_status   kp_device_info(int32_t device, int32_t* sm_count, int32_t* sm_clock_khz,
                           int32_t* cc);
/* Measured FP32 FMA-pipe throughput of the current device (TFLOP/s, best of
 * full-chip launches of scalar FFMA and packed FFMA2 chains at the clocks of
 * the moment): the K1 roofline peak. */
kp_status   kp_fp32_peak(double* tflops, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KP_ABI_H */
