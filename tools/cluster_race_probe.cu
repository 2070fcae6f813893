// Minimal 2-CTA cluster kernel with the same cluster barrier sequence as the
// tcgen05 CTA-pair kernel (barrier.cluster arrive.release / wait.acquire at
// start and end, nothing else in shared memory).  Run under
//   compute-sanitizer --tool racecheck --racecheck-report all ./cluster_race_probe
// to see whether the hazards racecheck reports for tc_gemm_pair_kernel at
// __shared__ 0x58-0x5f (below the kernel's dynamic shared memory, from a PC
// outside the kernel) come from the cluster barrier itself.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cluster_race_probe tools/cluster_race_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
                 ::: "memory");
}

// mode 0: cluster barriers only; mode 1: plus the pair kernel's TMEM
// allocation sequence (tcgen05.alloc / relinquish / dealloc with
// cta_group::2 by warp 1, an mbarrier initialised by warp 0 meanwhile).
__global__ void __cluster_dims__(2, 1, 1) probe(int* out, int mode) {
    extern __shared__ __align__(16) int smem[];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5;
    smem[threadIdx.x] = threadIdx.x;
    if (mode == 1 && warp == 0 && (threadIdx.x & 31) == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(
            uint32_t(__cvta_generic_to_shared(&bar))) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (mode == 1 && warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 64;"
                     :: "r"(uint32_t(__cvta_generic_to_shared(&tmem_slot))) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    cluster_sync();
    __syncthreads();
    int v = smem[(threadIdx.x + 1) % blockDim.x];
    const uint32_t tmem = mode == 1 ? tmem_slot : 0u;
    cluster_sync();
    if (mode == 1 && warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 64;" :: "r"(tmem) : "memory");
    if (v < 0) out[0] = v;
}

int main() {
    int* out;
    cudaMalloc(&out, 4);
    int rc = 0;
    for (int mode = 0; mode < 2; ++mode) {
        probe<<<148, 192, 4096>>>(out, mode);
        cudaError_t e = cudaDeviceSynchronize();
        std::printf("cluster probe mode %d: %s\n", mode, cudaGetErrorString(e));
        rc |= e != cudaSuccess;
    }
    return rc;
}
