// device_util.cuh -- small device helpers shared by the SentenceKV kernels.
#pragma once

#include <cuda_bf16.h>
#include <stdint.h>

namespace skv {

__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// 8 bf16 packed in a uint4 -> 8 fp32 (exact).
__device__ __forceinline__ void unpack8(const uint4& v, float* f) {
    f[0] = bf16lo(v.x); f[1] = bf16hi(v.x);
    f[2] = bf16lo(v.y); f[3] = bf16hi(v.y);
    f[4] = bf16lo(v.z); f[5] = bf16hi(v.z);
    f[6] = bf16lo(v.w); f[7] = bf16hi(v.w);
}

__device__ __forceinline__ uint32_t pack_bf16x2_rn(float lo, float hi) {
    __nv_bfloat16 a = __float2bfloat16_rn(lo), b = __float2bfloat16_rn(hi);
    return (uint32_t)__bfloat16_as_ushort(a) | ((uint32_t)__bfloat16_as_ushort(b) << 16);
}

// Streaming 128-bit global load (read once; do not allocate in L1).
__device__ __forceinline__ uint4 ld_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// Order-preserving fp32 -> u32 key (reading A14): -0 == +0, NaN -> 0 (ranks last).
__device__ __forceinline__ uint32_t ordered_key(float x) {
    if (x != x) return 0u;
    uint32_t u = __float_as_uint(x);
    if ((u & 0x7fffffffu) == 0u) u = 0u;
    return (u >> 31) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ bool in_set(int32_t tok, const int32_t* set, int n) {
    for (int i = 0; i < n; ++i)
        if (set[i] == tok) return true;
    return false;
}

// ---- block-wide scans (blockDim.x multiple of 32, <= 1024); `ws` = 32-entry smem workspace ----

template <typename T>
__device__ __forceinline__ T warp_incl_sum(T v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

// Inclusive sum over threads in index order; *total receives the block total.
template <typename T>
__device__ __forceinline__ T block_incl_sum(T v, T* ws, T* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_incl_sum(v);
    __syncthreads();  // protect ws from a previous use
    if (lane == 31) ws[warp] = v;
    __syncthreads();
    if (warp == 0) {
        T w = lane < nw ? ws[lane] : T(0);
        w = warp_incl_sum(w);
        if (lane < nw) ws[lane] = w;
    }
    __syncthreads();
    T base = warp > 0 ? ws[warp - 1] : T(0);
    *total = ws[nw - 1];
    return v + base;
}

__device__ __forceinline__ int warp_incl_max(int v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v = max(v, n);
    }
    return v;
}

// Exclusive max over threads in index order (identity `ident`).
__device__ __forceinline__ int block_excl_max(int v, int ident, int* ws) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int incl = warp_incl_max(v);
    __syncthreads();
    if (lane == 31) ws[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int w = lane < nw ? ws[lane] : ident;
        w = warp_incl_max(w);
        if (lane < nw) ws[lane] = w;
    }
    __syncthreads();
    int excl = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) excl = ident;
    if (warp > 0) excl = max(excl, ws[warp - 1]);
    return excl;
}

// ---- mbarrier + bulk async copy (TMA engine, non-tensor form) ----

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

// global -> shared bulk copy, completion counted in bytes on `bar`.  16-byte aligned, size % 16 == 0.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

// ---- deferred D1 state update (Eq. 2 sentence cache; reset at a boundary input, A11) ----
// Sq += q_t (or Sq = 0 when the step's input token is a boundary) for the grp query heads of unit
// (b, g), and its count.  Called by one CTA per unit after that unit's scoring and selection.
__device__ __forceinline__ void qs_update_unit(const __nv_bfloat16* __restrict__ q, const int32_t* __restrict__ input_token,
                               const int32_t* __restrict__ bset, int nb, float* __restrict__ Sq,
                               int32_t* __restrict__ cnt, int b, int g, int G, int grp, int D, int tid, int nthreads) {
    const bool reset = in_set(input_token[b], bset, nb);
    const size_t base = ((size_t)b * G * grp + (size_t)g * grp) * D;
    for (int i = tid; i < grp * D; i += nthreads)
        Sq[base + i] = reset ? 0.0f : __fadd_rn(Sq[base + i], __bfloat162float(q[base + i]));
    if (tid == 0) cnt[b * G + g] = reset ? 0 : cnt[b * G + g] + 1;
}

// ---- programmatic dependent launch (PDL) ----
// Every decode kernel is launched with programmatic stream serialization: it lets the next kernel
// of the stream start launching at once (trigger) and blocks until the previous kernel of the
// stream has completed and its writes are visible (wait) before reading any input.  Only
// input-independent setup (barrier init, smem carve-up) happens before the wait.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

}  // namespace skv

// ---- optional phase tracing (SKV_TRACE builds only): clock64 stamps of block (0,0,0), thread 0,
// into a per-translation-unit array `g_trace` that the file defines and exports for debugging ----
#ifdef SKV_TRACE
#define SKV_TRACE_DEFINE(name)                                                                  \
    __device__ long long g_trace[32];                                                           \
    extern "C" __attribute__((visibility("default"))) int sentencekv_debug_trace_##name(long long* out) { \
        return (int)cudaMemcpyFromSymbol(out, g_trace, sizeof(g_trace));                         \
    }
#define SKV_TRACE_POINT(slot)                                                                   \
    do {                                                                                        \
        if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0)          \
            g_trace[(slot)] = clock64();                                                        \
    } while (0)
#else
#define SKV_TRACE_DEFINE(name)
#define SKV_TRACE_POINT(slot) \
    do {                      \
    } while (0)
#endif
