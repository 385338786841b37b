// Does cp.async.bulk.prefetch.L2 make a later gather of the same runs hit L2?  Runs of ~7 KB (one
// selected sentence's K rows) at random offsets in a 1 GB buffer, 33 MB in total (one layer's
// selected K/V at 8b-128k).  Times the gather cold, after an L2-prefetch kernel, after a warming read.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

__global__ void gather(const uint4* __restrict__ buf, const long long* __restrict__ off, int nruns, int run16, float* sink) {
    uint32_t acc = 0;
    for (int r = blockIdx.x; r < nruns; r += gridDim.x) {
        const uint4* p = buf + off[r];
        for (int i = threadIdx.x; i < run16; i += blockDim.x) { uint4 v = p[i]; acc += v.x ^ v.w; }
    }
    if (acc == 12345u) sink[0] = acc;
}
__global__ void prefetch(const uint4* __restrict__ buf, const long long* __restrict__ off, int nruns, int bytes, int policy) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nruns) return;
    const void* p = buf + off[r];
    if (policy == 0) {
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
    } else {
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(p), "r"(bytes), "l"(pol) : "memory");
    }
}
__global__ void prefetch_ld(const uint4* __restrict__ buf, const long long* __restrict__ off, int nruns, int run16) {
    for (int r = blockIdx.x; r < nruns; r += gridDim.x) {
        const char* p = reinterpret_cast<const char*>(buf + off[r]);
        for (int i = threadIdx.x * 128; i < run16 * 16; i += blockDim.x * 128)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(p + i));
    }
}
__global__ void flushk(const uint4* p, size_t n, float* sink) {
    uint32_t acc = 0;
    for (size_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += (size_t)gridDim.x * 256) { uint4 v = p[i]; acc += v.y; }
    if (acc == 1u) sink[0] = acc;
}

int main() {
    const size_t total = 1ull << 30;
    const int run = 7168, run16 = run / 16, nruns = (33 << 20) / run;
    uint4* buf; float* sink; long long* doff;
    cudaMalloc(&buf, total); cudaMalloc(&sink, 4); cudaMalloc(&doff, nruns * 8);
    cudaMemset(buf, 1, total);
    std::mt19937_64 rng(1);
    std::vector<long long> off(nruns);
    for (auto& o : off) o = (long long)(rng() % ((total - run) / 256)) * 256 / 16;
    cudaMemcpy(doff, off.data(), nruns * 8, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto flush = [&] { flushk<<<1184, 256>>>(buf, total / 16, sink); };  // read 1 GB: L2 holds other data
    auto timed = [&](const char* name) {
        cudaEventRecord(a); gather<<<296, 256>>>(buf, doff, nruns, run16, sink); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); printf("%-40s %8.2f us\n", name, ms * 1e3);
    };
    for (int rep = 0; rep < 3; ++rep) {
        flush(); cudaDeviceSynchronize(); timed("cold gather");
        flush(); gather<<<296, 256>>>(buf, doff, nruns, run16, sink); cudaDeviceSynchronize(); timed("after warming gather");
        flush(); prefetch<<<(nruns + 255) / 256, 256>>>(buf, doff, nruns, run, 0); cudaDeviceSynchronize(); timed("after bulk prefetch.L2");
        flush(); prefetch<<<(nruns + 255) / 256, 256>>>(buf, doff, nruns, run, 1); cudaDeviceSynchronize(); timed("after bulk prefetch.L2 evict_last");
        flush(); prefetch_ld<<<296, 256>>>(buf, doff, nruns, run16); cudaDeviceSynchronize(); timed("after prefetch.global.L2 lines");
        // prefetch immediately followed by the gather (no sync): overlap
        flush(); cudaDeviceSynchronize();
        cudaEventRecord(a); prefetch<<<(nruns + 255) / 256, 256>>>(buf, doff, nruns, run, 0); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); printf("%-40s %8.2f us\n", "bulk prefetch kernel itself", ms * 1e3);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
