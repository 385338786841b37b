// prefill.cu -- P1 (sentence segmentation) and P2 (Eq. 1 sentence embeddings) on sm_100a.
//
// P1: PAPER.md P:391 (Sec. 4.1, "split the input text into sentences according to
//     punctuation"), P:430 (boundaries "e.g., period, question mark"), Alg. 1 line 2.
// P2: Eq. 1: kbar_{s,h} = (1/|S_s|) sum_{x in S_s} k_{x,h}; kept on the GPU.
#include "device_util.cuh"
#include "skv_internal.cuh"

namespace skv {

// One CTA per prompt.  Each thread owns a contiguous run of tokens.  Sentence ends are the
// boundary tokens (A1, A2), the last token (A4), and every tau-th token of a boundary-free run
// (A5 tau-cap).  Pass 1 finds the last boundary before each thread's run (block max-scan), pass
// 2 counts ends (block sum-scan -> sentence index base), pass 3 writes off[s+1] = end + 1.
__global__ void __launch_bounds__(1024) segment_kernel(const int32_t* __restrict__ tokens, int L,
                                                       const int32_t* __restrict__ bset, int nb, int tau,
                                                       int32_t* __restrict__ off, int off_stride,
                                                       int32_t* __restrict__ S_out, const int32_t* __restrict__ cap_b) {
    __shared__ int32_t sb[kMaxBoundary];
    __shared__ int32_t ws[32];
    const int b = blockIdx.x;
    // NEXT-3 outlier split: a per-prompt cap T below tau (reading A27); else the tau-cap (A5)
    if (cap_b) tau = min(tau, max(1, cap_b[b]));
    const int32_t* tok = tokens + (size_t)b * L;
    int32_t* o = off + (size_t)b * off_stride;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sb[i] = bset[i];
    __syncthreads();

    const int per = (L + blockDim.x - 1) / blockDim.x;
    const int lo = min(L, (int)threadIdx.x * per), hi = min(L, lo + per);

    int lastb = -1;
    for (int i = lo; i < hi; ++i)
        if (in_set(tok[i], sb, nb)) lastb = i;
    const int before = block_excl_max(lastb, -1, ws);

    int last = before, nend = 0;
    for (int i = lo; i < hi; ++i) {
        const bool bnd = in_set(tok[i], sb, nb);
        nend += (bnd || i == L - 1 || (i - last) % tau == 0) ? 1 : 0;
        if (bnd) last = i;
    }
    int total;
    const int base = block_incl_sum(nend, ws, &total) - nend;

    last = before;
    int k = base;
    for (int i = lo; i < hi; ++i) {
        const bool bnd = in_set(tok[i], sb, nb);
        if (bnd || i == L - 1 || (i - last) % tau == 0) o[++k] = i + 1;
        if (bnd) last = i;
    }
    if (threadIdx.x == 0) {
        o[0] = 0;
        S_out[b] = total;
    }
}

cudaError_t launch_segment(const int32_t* tokens, int B, int L, const int32_t* bset, int nb, int tau,
                           int32_t* off, int off_stride, int32_t* S, const int32_t* cap_b, cudaStream_t st) {
    segment_kernel<<<B, 1024, 0, st>>>(tokens, L, bset, nb, tau, off, off_stride, S, cap_b);
    return cudaGetLastError();
}

// One thread per (sentence, 8 dims): D/8 threads cover a sentence's key row (one 16-byte load
// per token), so a warp streams 2 (D=128) or 4 (D=64) sentences' contiguous K runs.  The sum is
// fp32 in ascending token order, then one IEEE division and bf16 round-to-nearest-even
// (canonical order A23; the oracle's skvref_embed states the same arithmetic independently).
template <int D>
__global__ void __launch_bounds__(256) compress_kernel(const __nv_bfloat16* __restrict__ K, int G, int L,
                                                       const int32_t* __restrict__ off, int off_stride,
                                                       const int32_t* __restrict__ S, int Smax,
                                                       __nv_bfloat16* __restrict__ E) {
    constexpr int LPS = D / 8;          // lanes per sentence
    constexpr int SPB = 256 / LPS;      // sentences per block
    constexpr int U = 4;                // loads in flight per thread
    const int b = blockIdx.z, g = blockIdx.y;
    const int s = blockIdx.x * SPB + threadIdx.x / LPS;
    const int lane = threadIdx.x % LPS;
    if (s >= S[b]) return;
    const int32_t* o = off + (size_t)b * off_stride;
    const int a = o[s], e = o[s + 1];
    const uint4* src = reinterpret_cast<const uint4*>(K + ((size_t)(b * G + g) * L) * D) + lane;
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
    int t = a;
    for (; t + U <= e; t += U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld_stream(src + (size_t)(t + u) * (D / 8));
#pragma unroll
        for (int u = 0; u < U; ++u) {
            float f[8];
            unpack8(v[u], f);
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = __fadd_rn(acc[i], f[i]);
        }
    }
    for (; t < e; ++t) {
        float f[8];
        unpack8(ld_stream(src + (size_t)t * (D / 8)), f);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = __fadd_rn(acc[i], f[i]);
    }
    const float n = (float)(e - a);
    uint4 out;
    out.x = pack_bf16x2_rn(__fdiv_rn(acc[0], n), __fdiv_rn(acc[1], n));
    out.y = pack_bf16x2_rn(__fdiv_rn(acc[2], n), __fdiv_rn(acc[3], n));
    out.z = pack_bf16x2_rn(__fdiv_rn(acc[4], n), __fdiv_rn(acc[5], n));
    out.w = pack_bf16x2_rn(__fdiv_rn(acc[6], n), __fdiv_rn(acc[7], n));
    reinterpret_cast<uint4*>(E + ((size_t)(b * G + g) * Smax + s) * D)[lane] = out;
}

cudaError_t launch_compress(const __nv_bfloat16* K, int B, int G, int L, int d, const int32_t* off,
                            int off_stride, const int32_t* S, int Smax, __nv_bfloat16* E, cudaStream_t st) {
    if (d == 128) {
        dim3 grid((Smax + 15) / 16, G, B);
        compress_kernel<128><<<grid, 256, 0, st>>>(K, G, L, off, off_stride, S, Smax, E);
    } else {
        dim3 grid((Smax + 31) / 32, G, B);
        compress_kernel<64><<<grid, 256, 0, st>>>(K, G, L, off, off_stride, S, Smax, E);
    }
    return cudaGetLastError();
}

}  // namespace skv
