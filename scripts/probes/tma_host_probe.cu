// Probe: can cp.async.bulk (TMA, non-tensor) read mapped pinned host memory, and what bandwidth do
// plain 128-bit loads from it reach?  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void bulk_from(const uint4* src, uint4* dst, int n16) {
    __shared__ alignas(128) uint4 buf[1024];
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const uint4* s = src + (size_t)blockIdx.x * 1024;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(16384));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(buf)),
                     "l"(s), "r"(16384), "r"(sa(&bar)) : "memory");
    }
    asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}" ::"r"(sa(&bar)) : "memory");
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) dst[(size_t)blockIdx.x * 1024 + i] = buf[i];
}

__global__ void ldg_from(const uint4* src, uint4* dst, size_t n16) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) dst[i] = src[i];
}

int main() {
    const size_t bytes = 1ull << 30, n16 = bytes / 16;
    uint4 *h, *hd, *d;
    cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
    cudaHostGetDevicePointer((void**)&hd, h, 0);
    for (size_t i = 0; i < n16; i += 997) h[i] = make_uint4(i, i + 1, i + 2, i + 3);
    cudaMalloc(&d, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float ms;
    // TMA bulk from host
    int blocks = (int)(n16 / 1024);
    bulk_from<<<blocks, 256>>>(hd, d, (int)n16);
    cudaError_t e = cudaDeviceSynchronize();
    printf("bulk_from_host: %s\n", cudaGetErrorString(e));
    if (e == cudaSuccess) {
        uint4 v; size_t i = 997 * 1000;
        cudaMemcpy(&v, d + i, 16, cudaMemcpyDeviceToHost);
        printf("check %s\n", (v.x == (uint32_t)i && v.w == (uint32_t)i + 3) ? "ok" : "MISMATCH");
        cudaEventRecord(a); bulk_from<<<blocks, 256>>>(hd, d, (int)n16); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b); printf("bulk_from_host GB/s %.1f\n", bytes / ms / 1e6);
    }
    cudaEventRecord(a); ldg_from<<<148 * 8, 256>>>(hd, d, n16); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("ldg_from_host GB/s %.1f (%s)\n", bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    cudaEventRecord(a); cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("memcpy H2D GB/s %.1f\n", bytes / ms / 1e6);
    cudaEventRecord(a); cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("memcpy D2H GB/s %.1f\n", bytes / ms / 1e6);
    return 0;
}
