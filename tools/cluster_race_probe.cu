// Minimal 2-CTA cluster kernel with the same cluster barrier sequence as the
// tcgen05 CTA-pair kernel (barrier.cluster arrive.release / wait.acquire at
// start and end, nothing else in shared memory).  Run under
//   compute-sanitizer --tool racecheck --racecheck-report all ./cluster_race_probe
// to see whether the hazards racecheck reports for tc_gemm_pair_kernel at
// __shared__ 0x58-0x5f (below the kernel's dynamic shared memory, from a PC
// outside the kernel) come from the cluster barrier itself.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cluster_race_probe tools/cluster_race_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
                 ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) probe(int* out) {
    extern __shared__ int smem[];
    smem[threadIdx.x] = threadIdx.x;
    cluster_sync();
    __syncthreads();
    int v = smem[(threadIdx.x + 1) % blockDim.x];
    cluster_sync();
    if (v < 0) out[0] = v;
}

int main() {
    int* out;
    cudaMalloc(&out, 4);
    probe<<<148, 192, 4096>>>(out);
    cudaError_t e = cudaDeviceSynchronize();
    std::printf("cluster probe: %s\n", cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}
