// Launch-gap probe: 32 back-to-back launches of an empty kernel shaped like the step kernel
// (256 CTAs in clusters of 8, 256 threads, ~100 KB dynamic smem) captured in a CUDA graph, with and
// without programmatic stream serialization.  Reports us per launch.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(256) empty_cluster(int* p) {
    extern __shared__ char sm[];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0 && p[0] == 12345) sm[0] = 1;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__global__ void __launch_bounds__(256) empty_plain(int* p) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0 && p[0] == 12345) p[1] = 1;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename K>
float run(K kernel, dim3 grid, size_t smem, bool pdl, cudaStream_t st, int* p) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 32; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid; cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = smem; cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
        cudaLaunchKernelEx(&cfg, kernel, p);
    }
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int i = 0; i < 5; ++i) cudaGraphLaunch(ge, st);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, st);
    for (int i = 0; i < 50; ++i) cudaGraphLaunch(ge, st);
    cudaEventRecord(b, st); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms * 1e3f / (50 * 32);
}

int main() {
    int* p; cudaMalloc(&p, 64); cudaMemset(p, 0, 64);
    cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    for (size_t smem : {0ul, 100ul << 10}) {
        for (bool pdl : {false, true}) {
            printf("cluster8 x256 CTAs smem %3zu KB pdl %d: %6.2f us/launch\n", smem >> 10, (int)pdl,
                   run(empty_cluster, dim3(8, 8, 4), smem, pdl, st, p));
            printf("plain    x256 CTAs smem %3zu KB pdl %d: %6.2f us/launch\n", smem >> 10, (int)pdl,
                   run(empty_plain, dim3(256), smem, pdl, st, p));
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
