// FP32 FFMA throughput microbenchmark: the measured denominator of the K1
// roofline (MEASURED_PEAKS.json carries only HBM and bf16 tensor peaks).
// Every thread runs 8 independent fma chains; a full-chip grid keeps all four
// SMSPs of every SM issuing back to back.  Two forms, the larger one wins:
// scalar FFMA with immediate operands (one register read per FMA) and the
// packed FFMA2 (fp32x2) form K1's inner product uses.
#include <algorithm>

#include "kp_internal.cuh"

namespace kp {

constexpr int kPeakChains = 8;
constexpr int kPeakIters = 8192;

__global__ void __launch_bounds__(256) ffma_peak_kernel(float* out, float seed) {
    float v[kPeakChains];
#pragma unroll
    for (int c = 0; c < kPeakChains; ++c) v[c] = seed + threadIdx.x * 1e-7f + c;
    const float b = 0.999999f, a = 1e-7f;
    for (int i = 0; i < kPeakIters; ++i) {
#pragma unroll
        for (int c = 0; c < kPeakChains; ++c) v[c] = fmaf(v[c], b, a);
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < kPeakChains; ++c) s += v[c];
    if (s == 123.456f) out[0] = s;  // keeps the chains live
}

__global__ void __launch_bounds__(256) ffma2_peak_kernel(float* out, float seed) {
    float2 v[kPeakChains];
#pragma unroll
    for (int c = 0; c < kPeakChains; ++c)
        v[c] = make_float2(seed + threadIdx.x * 1e-7f + c, seed - threadIdx.x * 1e-7f - c);
    const float2 b = make_float2(0.999999f, 0.999998f), a = make_float2(1e-7f, 2e-7f);
    for (int i = 0; i < kPeakIters / 2; ++i) {
#pragma unroll
        for (int c = 0; c < kPeakChains; ++c) v[c] = __ffma2_rn(v[c], b, a);
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < kPeakChains; ++c) s += v[c].x + v[c].y;
    if (s == 123.456f) out[0] = s;
}

}  // namespace kp

extern "C" kp_status kp_fp32_peak(double* tflops, void* stream_) {
    using namespace kp;
    if (!tflops) return fail(KP_ERR_INVALID_ARG, "null output");
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    float* scratch = nullptr;
    if (cudaMalloc(&scratch, sizeof(float)) != cudaSuccess) return check_launch("cudaMalloc");
    const dim3 grid(sms * 2), block(256);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0.0;
    for (int rep = 0; rep < 12; ++rep) {
        cudaEventRecord(e0, stream);
        if (rep % 2 == 0)
            ffma_peak_kernel<<<grid, block, 0, stream>>>(scratch, 1.0f + rep);
        else
            ffma2_peak_kernel<<<grid, block, 0, stream>>>(scratch, 1.0f + rep);
        note_launch();
        cudaEventRecord(e1, stream);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * kPeakChains * kPeakIters * double(grid.x) * block.x;
        if (rep > 1 && ms > 0.f) best = std::max(best, flops / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(scratch);
    kp_status st = check_launch("ffma_peak_kernel");
    if (st != KP_OK) return st;
    *tflops = best;
    return KP_OK;
}
