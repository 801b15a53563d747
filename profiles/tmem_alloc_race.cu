// tmem_alloc_race.cu -- minimal reproduction for the racecheck report on the
// tc pair kernel (profiles/sanitizer/r01_racecheck.log): a kernel that only
// allocates TMEM, publishes the address through the shared slot exactly as
// tc_gemm_kernel does (alloc -> tcgen05.fence::before_thread_sync -> CTA /
// cluster barrier -> tcgen05.fence::after_thread_sync -> read), and frees
// it.  No other shared-memory access exists in these kernels, so a hazard
// reported here comes from the tool's model of tcgen05.alloc alone.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tmem_race profiles/tmem_alloc_race.cu
//   compute-sanitizer --tool racecheck /tmp/tmem_race
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <int CTAS>
__global__ void __launch_bounds__(128, 1) alloc_only(uint32_t* out) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (warp == 1) {
        if constexpr (CTAS == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;\n" ::"r"(saddr(&slot)) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 64;\n" ::"r"(saddr(&slot)) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    if constexpr (CTAS == 2) cluster_sync(); else __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t base = slot;
    if (threadIdx.x == 0) out[blockIdx.x] = base;
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    if constexpr (CTAS == 2) cluster_sync(); else __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        if constexpr (CTAS == 1)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;\n" ::"r"(base) : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 64;\n" ::"r"(base) : "memory");
    }
}

int main() {
    uint32_t* d;
    cudaMalloc(&d, 64 * sizeof(uint32_t));
    alloc_only<1><<<4, 128>>>(d);
    printf("cta_group::1: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(4);
    cfg.blockDim = dim3(128);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, alloc_only<2>, d);
    printf("cta_group::2: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    uint32_t h[4];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("tmem bases: %u %u %u %u\n", h[0], h[1], h[2], h[3]);
    return 0;
}
