// variants.cu -- SURVEY 8(f) NEXT-3 (paper variants) and NEXT-4 (Quest pages) on the same D2-D4
// kernels (select_kernel, attend_mma_kernel):
//   NEXT-3 equal-size chunks        Sec. 6.1 "Sentence chunking", reading A26
//   NEXT-3 outlier split            App. "Effect of Sentence Length", reading A27
//   NEXT-3 current-token query      Sec. 6.2 -- a flag of the scoring kernels (qmode)
//   NEXT-3 skip-and-continue fill   alternative to the maximal prefix of P:444 (reading A13)
//   NEXT-4 Quest fixed pages        App. "Quest Sensitivity to Chunk Size", reading A28:
//                                   per-page min/max keys, bound sum_h sum_j max(q_j mn_j, q_j mx_j)
#include <cfloat>

#include "device_util.cuh"
#include "skv_internal.cuh"

namespace skv {
namespace {

// ---------------------------------------------------------------- outlier split threshold
// T = floor((L + n * sqrt(S * sum len^2 - L^2)) / S): mean + n * population std of the sentence
// lengths, from exact integer sums, in IEEE fp64 with every operation rounded separately (no
// contraction), the order the oracle's skvref_outlier_threshold writes.
__global__ void __launch_bounds__(256) outlier_cap_kernel(const int32_t* __restrict__ off, int off_stride,
                                                         const int32_t* __restrict__ S, double n,
                                                         int32_t* __restrict__ cap) {
    __shared__ unsigned long long ws[32];
    const int b = blockIdx.x;
    const int32_t* o = off + (size_t)b * off_stride;
    const int Sb = S[b];
    unsigned long long sq = 0;
    for (int s = threadIdx.x; s < Sb; s += blockDim.x) {
        const unsigned long long len = (unsigned long long)(o[s + 1] - o[s]);
        sq += len * len;
    }
    unsigned long long tot;
    block_incl_sum<unsigned long long>(sq, ws, &tot);
    if (threadIdx.x == 0) {
        const long long L = o[Sb] - o[0];
        const double var_s2 = (double)((long long)Sb * (long long)tot - L * L);
        double t = floor(__ddiv_rn(__dadd_rn((double)L, __dmul_rn(n, __dsqrt_rn(var_s2))), (double)Sb));
        t = fmin(fmax(t, 1.0), 2147483647.0);
        cap[b] = (int32_t)t;
    }
}

// ---------------------------------------------------------------- equal chunks / fixed pages
__global__ void __launch_bounds__(256) chunks_kernel(int L, int tau, int page, int32_t* __restrict__ off,
                                                    int off_stride, int32_t* __restrict__ S) {
    const int b = blockIdx.x;
    __shared__ int len_s;
    if (threadIdx.x == 0) {
        int len = page;
        if (len <= 0) {  // equal chunks: as many as the prompt has sentences, at most tau tokens each
            const int Sb = max(1, S[b]);
            len = min(tau, (L + Sb - 1) / Sb);
        }
        len_s = max(1, len);
    }
    __syncthreads();
    const int len = len_s, n = (L + len - 1) / len;
    int32_t* o = off + (size_t)b * off_stride;
    for (int k = threadIdx.x; k <= n; k += blockDim.x) o[k] = min(k * len, L);
    if (threadIdx.x == 0) S[b] = n;
}

// ---------------------------------------------------------------- Quest page metadata
// One thread per (page, 8 dims): elementwise min and max over the page's keys (exact, bf16 in and
// out; the first key seeds both, later ones replace on strict < / >, as skvref_quest_meta).
template <int D>
__global__ void __launch_bounds__(256) quest_meta_kernel(const __nv_bfloat16* __restrict__ K, int G, int L, int page,
                                                        const int32_t* __restrict__ S, int Smax,
                                                        __nv_bfloat16* __restrict__ E) {
    constexpr int LPS = D / 8;
    const int b = blockIdx.z, g = blockIdx.y;
    const int p = blockIdx.x * (256 / LPS) + threadIdx.x / LPS, l = threadIdx.x % LPS;
    if (p >= S[b]) return;
    const int a = p * page, e = min(L, a + page);
    const uint4* src = reinterpret_cast<const uint4*>(K + ((size_t)(b * G + g) * L) * D) + l;
    uint4 v = ld_stream(src + (size_t)a * LPS);
    float lo[8], hi[8];
    unpack8(v, lo);
    unpack8(v, hi);
    uint16_t lob[8], hib[8];
    const uint16_t* vb = reinterpret_cast<const uint16_t*>(&v);
#pragma unroll
    for (int i = 0; i < 8; ++i) lob[i] = hib[i] = vb[i];
    for (int t = a + 1; t < e; ++t) {
        const uint4 w = ld_stream(src + (size_t)t * LPS);
        float f[8];
        unpack8(w, f);
        const uint16_t* wb = reinterpret_cast<const uint16_t*>(&w);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (f[i] < lo[i]) { lo[i] = f[i]; lob[i] = wb[i]; }
            if (f[i] > hi[i]) { hi[i] = f[i]; hib[i] = wb[i]; }
        }
    }
    uint4 mn, mx;
    uint16_t* mnb = reinterpret_cast<uint16_t*>(&mn);
    uint16_t* mxb = reinterpret_cast<uint16_t*>(&mx);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        mnb[i] = lob[i];
        mxb[i] = hib[i];
    }
    uint4* dst = reinterpret_cast<uint4*>(E + (((size_t)(b * G + g) * Smax + p) * 2) * D);
    dst[l] = mn;
    dst[LPS + l] = mx;
}

// ---------------------------------------------------------------- Quest bounds (scores)
// Canonical fp32 order (A28): t_j = max(q_j*mn_j, q_j*mx_j) (exact bf16 x bf16 products, select
// a > b ? a : b); lane l of a page adds t[8l..8l+7] in order; the xor butterfly over the D/8 lanes
// (offsets D/16 .. 1) gives lane 0 the tree of the oracle; heads are summed in ascending order.
template <int D, int GRP>
__global__ void __launch_bounds__(256) quest_score_kernel(const __nv_bfloat16* __restrict__ q,
                                                         const __nv_bfloat16* __restrict__ E,
                                                         const int32_t* __restrict__ S, int G, int Smax,
                                                         float* __restrict__ scores) {
    constexpr int LPS = D / 8, PPB = 256 / LPS;
    __shared__ float qs[GRP][D];
    const int b = blockIdx.z, g = blockIdx.y;
    const int Hq = G * GRP;
    pdl_wait();
    for (int i = threadIdx.x; i < GRP * D; i += 256)
        qs[i / D][i % D] = __bfloat162float(q[((size_t)b * Hq + g * GRP) * D + i]);
    __syncthreads();
    const int p = blockIdx.x * PPB + threadIdx.x / LPS, l = threadIdx.x % LPS;
    const bool live = p < S[b];
    float mn[8], mx[8];
    if (live) {
        const uint4* src = reinterpret_cast<const uint4*>(E + (((size_t)(b * G + g) * Smax + p) * 2) * D);
        unpack8(src[l], mn);
        unpack8(src[LPS + l], mx);
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) mn[i] = mx[i] = 0.0f;
    }
    float U = 0.0f;
#pragma unroll
    for (int h = 0; h < GRP; ++h) {
        float acc = 0.0f;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float qj = qs[h][8 * l + i];
            const float a = __fmul_rn(qj, mn[i]), c = __fmul_rn(qj, mx[i]);
            const float t = a > c ? a : c;
            acc = i == 0 ? t : __fadd_rn(acc, t);
        }
#pragma unroll
        for (int o = LPS / 2; o >= 1; o >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
        U = h == 0 ? acc : __fadd_rn(U, acc);
    }
    if (live && l == 0) scores[(size_t)(b * G + g) * Smax + p] = U;
}

// ---------------------------------------------------------------- skip-and-continue fill
// On top of the prefix selection that select_kernel wrote into slot parity^1: repeatedly take the
// best-ranked unselected sentence that still fits the remaining budget (block max over key64 =
// (ordered(score) << 32) | ~s).  Since the budget only shrinks, this is the walk down the ranking
// that skips what does not fit.  Then one ordered compaction rewrites ids / offsets / sources.
constexpr int kSkThreads = 1024;

__global__ void __launch_bounds__(kSkThreads) skip_fill_kernel(const float* __restrict__ scores,
                                                              const int32_t* __restrict__ off, int off_stride,
                                                              const int32_t* __restrict__ S, int G, int Smax, int tau,
                                                              SelBufs sel, bool src_gathered,
                                                              int32_t* __restrict__ out_ids,
                                                              int32_t* __restrict__ out_count,
                                                              int32_t* __restrict__ out_tokens,
                                                              const int32_t* __restrict__ sid, int sid_stride) {
    extern __shared__ uint32_t bits[];  // [ceil(Smax / 32)] selected sentences
    __shared__ unsigned long long ws64[32];
    __shared__ unsigned long long s_best;
    __shared__ int s_rem;
    const int g = blockIdx.x, b = blockIdx.y, u = b * G + g, tid = threadIdx.x;
    const int Sb = S[b];
    const int32_t* o = off + (size_t)b * off_stride;
    const float* sc = scores + (size_t)u * Smax;
    const int cur = sel.parity[u] ^ 1;
    int32_t* ids = sel.ids_of(cur, u);
    int32_t* tokoff = sel.tok_of(cur, u);
    int32_t* src = sel.src_of(cur, u);
    const int nw = (Sb + 31) / 32;
    for (int i = tid; i < nw; i += kSkThreads) bits[i] = 0u;
    __syncthreads();
    const int count0 = *sel.count_of(cur, u);
    for (int i = tid; i < count0; i += kSkThreads) atomicOr(&bits[ids[i] >> 5], 1u << (ids[i] & 31));
    if (tid == 0) s_rem = tau - tokoff[count0];
    __syncthreads();
    for (;;) {
        const int rem = s_rem;
        unsigned long long best = 0ull;
        for (int s = tid; s < Sb; s += kSkThreads) {
            if ((bits[s >> 5] >> (s & 31)) & 1u) continue;
            if (o[s + 1] - o[s] > rem) continue;
            const unsigned long long k = ((unsigned long long)ordered_key(sc[s]) << 32) | (0xffffffffu - (uint32_t)s);
            best = k > best ? k : best;
        }
#pragma unroll
        for (int w = 16; w >= 1; w >>= 1) {
            const unsigned long long v = __shfl_xor_sync(0xffffffffu, best, w);
            best = v > best ? v : best;
        }
        if ((tid & 31) == 0) ws64[tid >> 5] = best;
        __syncthreads();
        if (tid == 0) {
            unsigned long long m = 0ull;
            for (int w = 0; w < kSkThreads / 32; ++w) m = ws64[w] > m ? ws64[w] : m;
            s_best = m;
            if (m) {
                const int s = (int)(0xffffffffu - (uint32_t)(m & 0xffffffffull));
                bits[s >> 5] |= 1u << (s & 31);
                s_rem = rem - (o[s + 1] - o[s]);
            }
        }
        __syncthreads();
        if (!s_best) break;
    }
    // ordered compaction over contiguous index ranges
    const int per = (Sb + kSkThreads - 1) / kSkThreads;
    const int i0 = min(Sb, tid * per), i1 = min(Sb, i0 + per);
    unsigned long long mine = 0;
    for (int s = i0; s < i1; ++s)
        if ((bits[s >> 5] >> (s & 31)) & 1u) mine += (1ull << 32) | (uint32_t)(o[s + 1] - o[s]);
    unsigned long long tot;
    const unsigned long long excl = block_incl_sum<unsigned long long>(mine, ws64, &tot) - mine;
    int pos = (int)(excl >> 32);
    uint32_t toff = (uint32_t)(excl & 0xffffffffull);
    for (int s = i0; s < i1; ++s) {
        if (!((bits[s >> 5] >> (s & 31)) & 1u)) continue;
        ids[pos] = s;
        tokoff[pos] = (int32_t)toff;
        src[pos] = src_gathered ? (int32_t)toff : o[s];
        if (out_ids) out_ids[(size_t)u * tau + pos] = sid ? sid[(size_t)b * sid_stride + s] : s;
        ++pos;
        toff += (uint32_t)(o[s + 1] - o[s]);
    }
    const int count = (int)(tot >> 32), ntok = (int)(tot & 0xffffffffull);
    if (tid == 0) {
        tokoff[count] = ntok;
        *sel.count_of(cur, u) = count;
        if (out_count) out_count[u] = count;
        if (out_tokens) out_tokens[u] = ntok;
    }
    if (out_ids)
        for (int i = count + tid; i < tau; i += kSkThreads) out_ids[(size_t)u * tau + i] = -1;
}

}  // namespace

cudaError_t launch_outlier_cap(const int32_t* off, int off_stride, const int32_t* S, int B, double n, int32_t* cap,
                               cudaStream_t st) {
    outlier_cap_kernel<<<B, 256, 0, st>>>(off, off_stride, S, n, cap);
    return cudaGetLastError();
}

cudaError_t launch_chunks(int B, int L, int tau, int page, int32_t* off, int off_stride, int32_t* S, cudaStream_t st) {
    chunks_kernel<<<B, 256, 0, st>>>(L, tau, page, off, off_stride, S);
    return cudaGetLastError();
}

cudaError_t launch_quest_meta(const __nv_bfloat16* K, int B, int G, int L, int d, int page, const int32_t* S, int Smax,
                              __nv_bfloat16* E, cudaStream_t st) {
    if (d == 128)
        quest_meta_kernel<128><<<dim3((Smax + 15) / 16, G, B), 256, 0, st>>>(K, G, L, page, S, Smax, E);
    else
        quest_meta_kernel<64><<<dim3((Smax + 31) / 32, G, B), 256, 0, st>>>(K, G, L, page, S, Smax, E);
    return cudaGetLastError();
}

cudaError_t launch_quest_score(const __nv_bfloat16* q, const __nv_bfloat16* E, const int32_t* S, int B, int G, int grp,
                               int d, int Smax, float* scores, cudaStream_t st) {
    const int ppb = 256 / (d / 8);
    const dim3 grid((Smax + ppb - 1) / ppb, G, B);
#define SKV_QS(DV, GV) return launch_pdl_if(false, quest_score_kernel<DV, GV>, grid, dim3(256), 0, st, q, E, S, G, Smax, scores)
    if (d == 128) {
        switch (grp) {
            case 1: SKV_QS(128, 1);
            case 2: SKV_QS(128, 2);
            case 4: SKV_QS(128, 4);
            case 8: SKV_QS(128, 8);
        }
    } else {
        switch (grp) {
            case 1: SKV_QS(64, 1);
            case 2: SKV_QS(64, 2);
            case 4: SKV_QS(64, 4);
            case 8: SKV_QS(64, 8);
        }
    }
#undef SKV_QS
    return cudaErrorInvalidValue;
}

cudaError_t launch_skip_fill(const float* scores, const int32_t* off, int off_stride, const int32_t* S, int B, int G,
                             int Smax, int tau, SelBufs sel, bool src_gathered, int32_t* out_ids, int32_t* out_count,
                             int32_t* out_tokens, const int32_t* sid, int sid_stride, cudaStream_t st) {
    const size_t smem = sizeof(uint32_t) * (size_t)((Smax + 31) / 32);
    cudaError_t e = ensure_smem((const void*)skip_fill_kernel, smem);
    if (e != cudaSuccess) return e;
    skip_fill_kernel<<<dim3(G, B), kSkThreads, smem, st>>>(scores, off, off_stride, S, G, Smax, tau, sel, src_gathered,
                                                          out_ids, out_count, out_tokens, sid, sid_stride);
    return cudaGetLastError();
}

}  // namespace skv
