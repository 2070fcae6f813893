// Host dispatch overhead of the compiled selectors (SURVEY §8(f) item 1:
// "measure host dispatch overhead, target < 1 us").
//
//   g++ -O2 -std=c++17 -I include tools/dispatch_bench.cpp \
//       -L paper_2003_06795_b200 -lkp -Wl,-rpath,$PWD/paper_2003_06795_b200 \
//       -I /usr/local/cuda/include -L /usr/local/cuda/lib64 -lcudart -o /tmp/dispatch_bench
//
// Part 1 (no GPU needed): ns per kp_select call (decision-tree walk + the
// selector table lookup) over 4096 log-uniform shapes, per family/variant.
// Part 2 (GPU): host-side enqueue cost of kp_gemm_auto vs kp_gemm with the
// same config on a small problem -- the difference is the dispatch overhead
// a caller pays on top of the launch itself.  Prints one JSON line.
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "kp_abi.h"

using clk = std::chrono::steady_clock;

// the parameter bytes of a tcgen05 launch: three 128-byte tensor maps + TcParams
struct ParamBlob {
    unsigned char bytes[3 * 128 + 96];
};
__global__ void empty_kernel(ParamBlob) {}

int main() {
    std::mt19937_64 rng(7);
    std::uniform_real_distribution<double> u(0.0, std::log(8192.0));
    std::vector<int64_t> shapes(3 * 4096);
    for (auto& v : shapes) v = std::max<int64_t>(1, int64_t(std::exp(u(rng))));
    std::printf("{\"select_ns\": {");
    const char* fams[] = {"f32", "tf32", "bf16"};
    bool first = true;
    for (int f = 0; f < 3; ++f)
        for (int lay = 0; lay < 4; ++lay) {
            const int ta = lay >> 1, tb = lay & 1;
            kp_config c;
            if (kp_select(kp_family(f), ta, tb, 64, 64, 64, &c) != KP_OK) continue;
            const int iters = 4'000'000;
            uint32_t sink = 0;
            auto t0 = clk::now();
            for (int i = 0; i < iters; ++i) {
                const int64_t* s = &shapes[3 * (i & 4095)];
                kp_select(kp_family(f), ta, tb, s[0], s[1], s[2], &c);
                sink += c.acc;
            }
            double ns = std::chrono::duration<double, std::nano>(clk::now() - t0).count() / iters;
            static const char* lays[] = {"nn", "nt", "tn", "tt"};
            std::printf("%s\"%s_%s\": %.1f", first ? "" : ", ", fams[f], lays[lay], ns);
            first = false;
            if (sink == 0xFFFFFFFF) std::printf(" ");
        }
    std::printf("}");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        std::printf(", \"enqueue_us\": null}\n");
        return 0;
    }
    const int64_t m = 128, k = 128, n = 128;
    float *A, *B, *C;
    cudaMalloc(&A, m * k * 4);
    cudaMalloc(&B, k * n * 4);
    cudaMalloc(&C, m * n * 4);
    cudaStream_t s;
    cudaStreamCreate(&s);
    kp_gemm_desc d = {1, m, k, n, 0, 0, k, n, n, 0, 0, 0, 1.0f, 0.0f};
    kp_config cfg;
    kp_select(KP_F32_SIMT, 0, 0, m, k, n, &cfg);
    double direct = 1e30, autod = 1e30;
    for (int rep = 0; rep < 5; ++rep) {
        for (int mode = 0; mode < 2; ++mode) {
            const int iters = 2000;
            cudaStreamSynchronize(s);
            auto t0 = clk::now();
            for (int i = 0; i < iters; ++i) {
                if (mode == 0) kp_gemm(KP_F32_SIMT, cfg, &d, A, B, C, s);
                else kp_gemm_auto(KP_F32_SIMT, &d, A, B, C, s, nullptr);
                if ((i & 255) == 255) cudaStreamSynchronize(s);  // bound the queue
            }
            double us = std::chrono::duration<double, std::micro>(clk::now() - t0).count() / iters;
            (mode == 0 ? direct : autod) = std::min(mode == 0 ? direct : autod, us);
        }
    }
    cudaStreamSynchronize(s);
    std::printf(", \"enqueue_us\": {\"kp_gemm\": %.3f, \"kp_gemm_auto\": %.3f, "
                "\"auto_minus_direct\": %.3f, \"problem\": [%ld, %ld, %ld]}",
                direct, autod, autod - direct, long(m), long(k), long(n));
    // tcgen05 launch (BF16 256^3, one tile per CTA, no split) against a bare
    // launch of an empty kernel carrying the same parameter bytes: host time
    // of the enqueue calls only (the stream is drained between batches of 32,
    // outside the timed spans) -- the library's share of the host enqueue
    const int64_t t = 256;
    void *A2, *B2;
    float* C2;
    cudaMalloc(&A2, t * t * 2);
    cudaMalloc(&B2, t * t * 2);
    cudaMalloc(&C2, t * t * 4);
    kp_gemm_desc d2 = {1, t, t, t, 0, 0, t, t, t, 0, 0, 0, 1.0f, 0.0f};
    const kp_config tc = {1, 1, 4, 8, 8};
    kp_set_tc_split(0);
    double tc_us = 1e30, bare_us = 1e30;
    for (int rep = 0; rep < 5; ++rep) {
        double tsum = 0.0, bsum = 0.0;
        for (int batch = 0; batch < 16; ++batch) {
            cudaStreamSynchronize(s);
            auto t0 = clk::now();
            for (int i = 0; i < 32; ++i) kp_gemm(KP_BF16_TC, tc, &d2, A2, B2, C2, s);
            tsum += std::chrono::duration<double, std::micro>(clk::now() - t0).count();
            cudaStreamSynchronize(s);
            t0 = clk::now();
            for (int i = 0; i < 32; ++i) empty_kernel<<<4, 192, 0, s>>>(ParamBlob{});
            bsum += std::chrono::duration<double, std::micro>(clk::now() - t0).count();
        }
        tc_us = std::min(tc_us, tsum / 512);
        bare_us = std::min(bare_us, bsum / 512);
    }
    kp_set_tc_split(1);
    cudaStreamSynchronize(s);
    std::printf(", \"tc_enqueue_us\": {\"kp_gemm_bf16_256\": %.3f, \"bare_launch_same_param_bytes\": %.3f, "
                "\"note\": \"host time of the enqueue calls only\"}}\n",
                tc_us, bare_us);
    return 0;
}
