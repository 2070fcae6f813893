// FFMA issue-rate probe (investigation tool, not part of libkp): what fraction
// of the FFMA peak can a register-tiled GEMM inner loop reach at all on this
// part?  Three kernels, full chip (2 CTAs x 256 threads per SM, like K1):
//   imm   : v = fma(v, c1, c2)              (the kp_fp32_peak pattern)
//   reg   : acc[i][j] = fma(a[i], b[j], acc[i][j]), a/b in registers (8x8)
//   lds   : the same 8x8 outer product with a/b re-read from shared memory
//           every k (LDS.128 x4 per 64 FFMA, K1's acc=4 mix), no global traffic
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma_probe tools/ffma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void __launch_bounds__(256, 2) k_imm(float* out, float s) {
    float v[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = s + threadIdx.x * 1e-7f + c;
    for (int i = 0; i < ITERS * 8; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) v[c] = fmaf(v[c], 0.999999f, 1e-7f);
    }
    float t = 0.f;
#pragma unroll
    for (int c = 0; c < 8; ++c) t += v[c];
    if (t == 123.456f) out[0] = t;
}

__global__ void __launch_bounds__(256, 2) k_reg(float* out, float s) {
    float a[8], b[8], acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = s + i * 1e-3f + threadIdx.x * 1e-7f; b[i] = s - i * 1e-3f; }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) t += acc[i][j];
    if (t == 123.456f) out[0] = t;
}

__global__ void __launch_bounds__(256, 2) k_lds(float* out, float s) {
    __shared__ __align__(16) float sm[2][32][4 * 8 + 4];
    for (int i = threadIdx.x; i < 2 * 32 * 36; i += blockDim.x) (&sm[0][0][0])[i] = s + i * 1e-6f;
    __syncthreads();
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    const int ta = threadIdx.x & 7, tb = (threadIdx.x >> 3) & 3;
    for (int it = 0; it < ITERS / 32; ++it) {
#pragma unroll 4
        for (int k = 0; k < 32; ++k) {
            const float4 a0 = *reinterpret_cast<const float4*>(&sm[0][k][ta * 4]);
            const float4 a1 = *reinterpret_cast<const float4*>(&sm[0][(k + 1) & 31][ta * 4]);
            const float4 b0 = *reinterpret_cast<const float4*>(&sm[1][k][tb * 8]);
            const float4 b1 = *reinterpret_cast<const float4*>(&sm[1][k][tb * 8 + 4]);
            float a[8], b[8];
            a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
            a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
            b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
            b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
    }
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) t += acc[i][j];
    if (t == 123.456f) out[0] = t;
}

// FFMA2 (sm_100 packed fp32x2, __ffma2_rn): acc pairs along the column axis,
// the row operand broadcast -- ptxas folds make_float2(a, a) into the
// FFMA2 scalar-operand form, so an 8x8 outer product is 32 instructions.
__global__ void __launch_bounds__(256, 2) k_reg2(float* out, float s) {
    float a[8];
    float2 b[4], acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = s + i * 1e-3f + threadIdx.x * 1e-7f;
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = make_float2(s - j * 1e-3f, s + j * 1e-3f);
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = __ffma2_rn(make_float2(a[i], a[i]), b[j], acc[i][j]);
    }
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) t += acc[i][j].x + acc[i][j].y;
    if (t == 123.456f) out[0] = t;
}

__global__ void __launch_bounds__(256, 2) k_lds2(float* out, float s) {
    __shared__ __align__(16) float sm[2][32][4 * 8 + 4];
    for (int i = threadIdx.x; i < 2 * 32 * 36; i += blockDim.x) (&sm[0][0][0])[i] = s + i * 1e-6f;
    __syncthreads();
    float2 acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
    const int ta = threadIdx.x & 7, tb = (threadIdx.x >> 3) & 3;
    for (int it = 0; it < ITERS / 32; ++it) {
#pragma unroll 4
        for (int k = 0; k < 32; ++k) {
            const float4 a0 = *reinterpret_cast<const float4*>(&sm[0][k][ta * 4]);
            const float4 a1 = *reinterpret_cast<const float4*>(&sm[0][(k + 1) & 31][ta * 4]);
            const float4 b0 = *reinterpret_cast<const float4*>(&sm[1][k][tb * 8]);
            const float4 b1 = *reinterpret_cast<const float4*>(&sm[1][k][tb * 8 + 4]);
            float a[8];
            a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
            a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
            float2 b[4];
            b[0] = make_float2(b0.x, b0.y); b[1] = make_float2(b0.z, b0.w);
            b[2] = make_float2(b1.x, b1.y); b[3] = make_float2(b1.z, b1.w);
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = __ffma2_rn(make_float2(a[i], a[i]), b[j], acc[i][j]);
        }
    }
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) t += acc[i][j].x + acc[i][j].y;
    if (t == 123.456f) out[0] = t;
}

template <typename F>
static void run(const char* name, F kern, double flops_per_thread) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* d;
    cudaMalloc(&d, 4);
    const dim3 grid(sms * 2), block(256);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0;
    for (int r = 0; r < 6; ++r) {
        cudaEventRecord(e0);
        kern<<<grid, block>>>(d, 1.0f + r);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double tf = flops_per_thread * grid.x * block.x / (ms * 1e-3) / 1e12;
        if (r > 0 && tf > best) best = tf;
    }
    printf("{\"probe\": \"%s\", \"tflops\": %.2f, \"err\": \"%s\"}\n", name, best,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    run("imm", k_imm, 2.0 * 8 * 8 * ITERS);
    run("reg8x8", k_reg, 2.0 * 64 * ITERS);
    run("lds8x8", k_lds, 2.0 * 64 * ITERS);
    run("reg8x8_ffma2", k_reg2, 2.0 * 64 * ITERS);
    run("lds8x8_ffma2", k_lds2, 2.0 * 64 * ITERS);
    return 0;
}
