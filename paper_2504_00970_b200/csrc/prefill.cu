// prefill.cu -- P1 (sentence segmentation) and P2 (Eq. 1 sentence embeddings) on sm_100a.
//
// P1: PAPER.md P:391 (Sec. 4.1, "split the input text into sentences according to
//     punctuation"), P:430 (boundaries "e.g., period, question mark"), Alg. 1 line 2.
// P2: Eq. 1: kbar_{s,h} = (1/|S_s|) sum_{x in S_s} k_{x,h}; kept on the GPU.
#include "device_util.cuh"
#include "skv_internal.cuh"

namespace skv {

// P1 segmentation, multi-CTA (r02; the r01 kernel used one CTA per prompt and ran at 6.6 GB/s,
// 0.32 ms for 4 x 131072 tokens).  Chunks of kSegChunk tokens, one CTA each, thread = 8 consecutive tokens;
// the boundary set is sorted on the host, membership by binary search.  Same rules and output as
// segment_kernel: a sentence ends at a boundary token, at L-1, or every tau-th token of a
// boundary-free run (the tau-cap counts from the last boundary, so only the last boundary before
// each token is carried across chunks):
//   seg_lastb_kernel: last boundary of every chunk;
//   seg_count_kernel: ends per chunk (last boundary before the chunk = max over the chunks before);
//   seg_write_kernel: offsets (base = ends of the chunks before + a block scan).
constexpr int kSegThreads = 256, kSegPer = 8, kSegChunk = kSegThreads * kSegPer;

__device__ __forceinline__ bool in_sorted(int32_t tok, const int32_t* set, int n) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (set[mid] < tok) lo = mid + 1; else hi = mid;
    }
    return lo < n && set[lo] == tok;
}

__global__ void __launch_bounds__(kSegThreads) seg_lastb_kernel(const int32_t* __restrict__ tokens, int L,
                                                               const int32_t* __restrict__ bset, int nb,
                                                               int32_t* __restrict__ lastb) {
    __shared__ int32_t sb[kMaxBoundary];
    __shared__ int ws[32];
    const int b = blockIdx.y, c = blockIdx.x;
    for (int i = threadIdx.x; i < nb; i += kSegThreads) sb[i] = bset[i];
    __syncthreads();
    const int32_t* tok = tokens + (size_t)b * L;
    int lb = -1;
    for (int i = c * kSegChunk + threadIdx.x; i < min(L, (c + 1) * kSegChunk); i += kSegThreads)
        if (in_sorted(tok[i], sb, nb)) lb = max(lb, i);
    lb = __reduce_max_sync(0xffffffffu, lb);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = lb;
    __syncthreads();
    if (threadIdx.x == 0) {
        int m = -1;
        for (int w = 0; w < kSegThreads / 32; ++w) m = max(m, ws[w]);
        lastb[(size_t)b * gridDim.x + c] = m;
    }
}

// per thread: its 8 tokens' boundary flags and the last boundary before them; returns the ends
template <bool WRITE>
__device__ __forceinline__ int seg_chunk(const int32_t* tok, int L, const int32_t* sb, int nb, int tau, int c,
                                         int lastb_in, int* ws, int32_t* o, int base) {
    const int i0 = c * kSegChunk + threadIdx.x * kSegPer;
    bool bnd[kSegPer];
    int lb = -1;
#pragma unroll
    for (int u = 0; u < kSegPer; ++u) {
        const int i = i0 + u;
        bnd[u] = i < L && in_sorted(tok[i], sb, nb);
        if (bnd[u]) lb = i;
    }
    int before = block_excl_max(lb, -1, ws);
    before = max(before, lastb_in);
    int last = before, n = 0;
#pragma unroll
    for (int u = 0; u < kSegPer; ++u) {
        const int i = i0 + u;
        if (i < L && (bnd[u] || i == L - 1 || (i - last) % tau == 0)) ++n;
        if (bnd[u]) last = i;
    }
    if constexpr (WRITE) {
        int total;
        int k = base + block_incl_sum(n, ws, &total) - n;
        last = before;
#pragma unroll
        for (int u = 0; u < kSegPer; ++u) {
            const int i = i0 + u;
            if (i < L && (bnd[u] || i == L - 1 || (i - last) % tau == 0)) o[++k] = i + 1;
            if (bnd[u]) last = i;
        }
        return total;
    } else {
        int total;
        block_incl_sum(n, ws, &total);
        return total;
    }
}

__global__ void __launch_bounds__(kSegThreads) seg_count_kernel(const int32_t* __restrict__ tokens, int L,
                                                               const int32_t* __restrict__ bset, int nb, int tau,
                                                               const int32_t* __restrict__ cap_b,
                                                               const int32_t* __restrict__ lastb,
                                                               int32_t* __restrict__ ends) {
    __shared__ int32_t sb[kMaxBoundary];
    __shared__ int ws[32];
    __shared__ int s_in;
    const int b = blockIdx.y, c = blockIdx.x, nch = gridDim.x;
    if (cap_b) tau = min(tau, max(1, cap_b[b]));
    for (int i = threadIdx.x; i < nb; i += kSegThreads) sb[i] = bset[i];
    if (threadIdx.x < 32) {
        int m = -1;
        for (int x = threadIdx.x; x < c; x += 32) m = max(m, lastb[(size_t)b * nch + x]);
        m = __reduce_max_sync(0xffffffffu, m);
        if (threadIdx.x == 0) s_in = m;
    }
    __syncthreads();
    const int total = seg_chunk<false>(tokens + (size_t)b * L, L, sb, nb, tau, c, s_in, ws, nullptr, 0);
    if (threadIdx.x == 0) ends[(size_t)b * nch + c] = total;
}

__global__ void __launch_bounds__(kSegThreads) seg_write_kernel(const int32_t* __restrict__ tokens, int L,
                                                               const int32_t* __restrict__ bset, int nb, int tau,
                                                               const int32_t* __restrict__ cap_b,
                                                               const int32_t* __restrict__ lastb,
                                                               const int32_t* __restrict__ ends,
                                                               int32_t* __restrict__ off, int off_stride,
                                                               int32_t* __restrict__ S_out) {
    __shared__ int32_t sb[kMaxBoundary];
    __shared__ int ws[32];
    __shared__ int s_in, s_base;
    const int b = blockIdx.y, c = blockIdx.x, nch = gridDim.x;
    if (cap_b) tau = min(tau, max(1, cap_b[b]));
    for (int i = threadIdx.x; i < nb; i += kSegThreads) sb[i] = bset[i];
    if (threadIdx.x < 32) {
        int m = -1, e = 0;
        for (int x = threadIdx.x; x < c; x += 32) {
            m = max(m, lastb[(size_t)b * nch + x]);
            e += ends[(size_t)b * nch + x];
        }
        m = __reduce_max_sync(0xffffffffu, m);
        e = __reduce_add_sync(0xffffffffu, e);
        if (threadIdx.x == 0) {
            s_in = m;
            s_base = e;
        }
    }
    __syncthreads();
    int32_t* o = off + (size_t)b * off_stride;
    const int total = seg_chunk<true>(tokens + (size_t)b * L, L, sb, nb, tau, c, s_in, ws, o, s_base);
    if (threadIdx.x == 0 && c == nch - 1) {
        o[0] = 0;
        S_out[b] = s_base + total;
    }
}

cudaError_t launch_segment(const int32_t* tokens, int B, int L, const int32_t* bset, int nb, int tau,
                           int32_t* off, int off_stride, int32_t* S, const int32_t* cap_b, int32_t* scratch,
                           cudaStream_t st) {
    const int nch = (L + kSegChunk - 1) / kSegChunk;
    int32_t* lastb = scratch;             // [B][nch]
    int32_t* ends = scratch + (size_t)B * nch;  // [B][nch]
    seg_lastb_kernel<<<dim3(nch, B), kSegThreads, 0, st>>>(tokens, L, bset, nb, lastb);
    seg_count_kernel<<<dim3(nch, B), kSegThreads, 0, st>>>(tokens, L, bset, nb, tau, cap_b, lastb, ends);
    seg_write_kernel<<<dim3(nch, B), kSegThreads, 0, st>>>(tokens, L, bset, nb, tau, cap_b, lastb, ends, off,
                                                          off_stride, S);
    return cudaGetLastError();
}

size_t segment_scratch_ints(int B, int L) { return 2 * (size_t)B * ((L + kSegChunk - 1) / kSegChunk); }

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
