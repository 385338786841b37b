// decode_select.cu -- D1 (Eq. 2 sentence query cache + similarity scoring) and D2 (budgeted
// whole-sentence selection) on sm_100a.
//
// D1: Eq. 2, PAPER.md P:431-435 (qbar = mean of the sentence cache Q_s); similarity
//     S(qbar, kbar_{s,h}) = qbar^T kbar_{s,h} for every sentence bucket;
//     Alg. 1 lines 14-16.  Reset of Q_s at a boundary: Alg. 1 l.19-21.
// D2: "rank all sentence buckets by their similarity scores and retrieve tokens from the most
//     relevant buckets in descending order ... until we reach our token budget",
//     Alg. 1 line 17.  Readings A9-A15, A23.
#include "device_util.cuh"
#include "skv_internal.cuh"

namespace skv {

// ------------------------------------------------------------------------------ D1 scoring
//
// Grid (splits, G, B); each CTA scores a contiguous range of sentences of one (b, g) unit.
// Every CTA forms qt_g = sum_h qbar_h with qbar_h = (Sq_h + q_h) / (cnt + 1) (the appended,
// not yet stored, Q_s of this step; the state itself is written by the select kernel, which
// runs after all scoring CTAs).  Then D/8 lanes per sentence: lane l holds qt[8l..8l+7] in
// registers and reads one 16-byte chunk of the sentence embedding; the fp32 dot follows the
// canonical order (mul, 7 fma, then xor-butterfly adds whose lane-0 result equals the tree of
// A23).  E is read exactly once per step: the HBM-bound part of decode.
template <int D>
__global__ void __launch_bounds__(256) score_kernel(const __nv_bfloat16* __restrict__ q,
                                                    const float* __restrict__ Sq, const int32_t* __restrict__ cnt,
                                                    const __nv_bfloat16* __restrict__ E,
                                                    const int32_t* __restrict__ S, int G, int grp, int Smax,
                                                    int chunk, float* __restrict__ scores) {
    constexpr int LPS = D / 8;
    constexpr int GPW = 32 / LPS;  // sentence groups per warp
    constexpr int U = 4;           // sentences in flight per lane group
    __shared__ float qt[D];
    const int b = blockIdx.z, g = blockIdx.y;
    const int Sb = S[b];
    const int s0 = blockIdx.x * chunk;
    if (s0 >= Sb) return;
    const int s1 = min(Sb, s0 + chunk);
    const int Hq = G * grp;

    const float c = (float)(cnt[b] + 1);
    for (int j = threadIdx.x; j < D; j += blockDim.x) {
        float acc = 0.0f;
        for (int h = 0; h < grp; ++h) {
            const size_t idx = ((size_t)b * Hq + g * grp + h) * D + j;
            const float v = __fadd_rn(Sq[idx], __bfloat162float(q[idx]));
            const float qb = __fdiv_rn(v, c);
            acc = (h == 0) ? qb : __fadd_rn(acc, qb);
        }
        qt[j] = acc;
    }
    __syncthreads();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int l = lane % LPS, grp_in_warp = lane / LPS;
    float qr[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) qr[i] = qt[8 * l + i];

    const uint4* Eu = reinterpret_cast<const uint4*>(E + (size_t)(b * G + g) * Smax * D);
    float* out = scores + (size_t)(b * G + g) * Smax;
    const int nwarps = blockDim.x >> 5;
    // warp-uniform loop: every lane takes part in every shuffle
    for (int base = s0 + warp * GPW * U; base < s1; base += nwarps * GPW * U) {
        uint4 e[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int s = base + u * GPW + grp_in_warp;
            e[u] = s < s1 ? ld_stream(Eu + (size_t)s * LPS + l) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            float f[8];
            unpack8(e[u], f);
            float p = __fmul_rn(qr[0], f[0]);
#pragma unroll
            for (int i = 1; i < 8; ++i) p = __fmaf_rn(qr[i], f[i], p);
#pragma unroll
            for (int o = LPS / 2; o >= 1; o >>= 1) p = __fadd_rn(p, __shfl_xor_sync(0xffffffffu, p, o));
            const int s = base + u * GPW + grp_in_warp;
            if (l == 0 && s < s1) out[s] = p;
        }
    }
}

cudaError_t launch_score(const __nv_bfloat16* q, const float* Sq, const int32_t* cnt, const __nv_bfloat16* E,
                         const int32_t* S, int B, int G, int grp, int d, int Smax, float* scores,
                         cudaStream_t st) {
    // Fill ~2 waves of 148 SMs: split each (b, g) unit's sentences into `splits` ranges.
    const int units = B * G;
    int splits = (2 * kNumSMs + units - 1) / units;
    int chunk = (Smax + splits - 1) / splits;
    chunk = max(64, (chunk + 63) / 64 * 64);
    splits = (Smax + chunk - 1) / chunk;
    dim3 grid(splits, G, B);
    if (d == 128)
        score_kernel<128><<<grid, 256, 0, st>>>(q, Sq, cnt, E, S, G, grp, Smax, chunk, scores);
    else
        score_kernel<64><<<grid, 256, 0, st>>>(q, Sq, cnt, E, S, G, grp, Smax, chunk, scores);
    return cudaGetLastError();
}

// ----------------------------------------------------------------------------- D2 selection
//
// One CTA (1024 threads) per (b, g).  The selection is the maximal prefix of the ranking by
// key = (ordered(score), -index) whose token count fits tau (A13, A14).  Equivalently: find
// the first sentence s* (in rank order) at which the cumulative length exceeds tau; select
// every sentence ranked before it.  s* is found by a length-weighted radix select on the
// 32-bit ordered score (digits 11/11/10 bits; each pass histograms the lengths of the
// sentences whose key matches the prefix found so far, then one block scan locates the bin
// where the cumulative length from the top crosses the remaining budget).  If that bin holds
// one sentence it is s*; if the full 32-bit key is reached with several tied sentences, s* is
// located among them in ascending index order (the tie rule) by an ordered block scan.  A last
// ordered pass compacts the selected ids in ascending order with their token prefix sums.
//
// The same CTA performs the deferred D1 state update of its query heads: Sq += q_t, or Sq = 0
// when the step's input token is a boundary (A11); cnt is updated by the g == 0 CTA.
constexpr int kSelThreads = 1024;
constexpr int kBins = 2048;

__global__ void __launch_bounds__(kSelThreads) select_kernel(
    const float* __restrict__ scores, const int32_t* __restrict__ off, int off_stride,
    const int32_t* __restrict__ S, int G, int grp, int D, int Smax, int tau, const __nv_bfloat16* __restrict__ q,
    const int32_t* __restrict__ input_token, const int32_t* __restrict__ bset, int nb, float* __restrict__ Sq,
    int32_t* __restrict__ cnt, int32_t* __restrict__ sel_ids, int32_t* __restrict__ sel_tokoff,
    int32_t* __restrict__ sel_count, int32_t* __restrict__ out_ids, int32_t* __restrict__ out_count,
    int32_t* __restrict__ out_tokens) {
    __shared__ uint32_t hw[kBins];  // length-weighted histogram
    __shared__ uint32_t hc[kBins];  // count histogram
    __shared__ uint32_t ws32[32];
    __shared__ unsigned long long ws64[32];
    __shared__ uint32_t sh_bin, sh_rem, sh_cnt;
    __shared__ int sh_found;

    const int g = blockIdx.x, b = blockIdx.y;
    const int tid = threadIdx.x;
    const int Sb = S[b];
    const float* sc = scores + (size_t)(b * G + g) * Smax;
    const int32_t* o = off + (size_t)b * off_stride;
    const int Hq = G * grp;

    // ---- deferred D1 state update (Eq. 2 sentence cache; reset at a boundary input) ----
    {
        const bool reset = in_set(input_token[b], bset, nb);
        const size_t base = ((size_t)b * Hq + (size_t)g * grp) * D;
        for (int i = tid; i < grp * D; i += blockDim.x)
            Sq[base + i] = reset ? 0.0f : __fadd_rn(Sq[base + i], __bfloat162float(q[base + i]));
        if (g == 0 && tid == 0) cnt[b] = reset ? 0 : cnt[b] + 1;
    }

    // ---- radix select for the crossing key ----
    uint32_t prefix = 0, mask = 0, rem = (uint32_t)tau;
    bool all_fit = false, resolved = false;
    const int shifts[3] = {21, 10, 0};
    const int widths[3] = {11, 11, 10};
    for (int pass = 0; pass < 3 && !resolved; ++pass) {
        const int shift = shifts[pass];
        const uint32_t dmask = (1u << widths[pass]) - 1u;
        for (int i = tid; i < kBins; i += blockDim.x) hw[i] = hc[i] = 0u;
        __syncthreads();
        // warp-uniform trip count; lanes whose sentence falls in the same bin are aggregated
        // (match_any + reduce) so concentrated score distributions do not serialise on one
        // shared-memory address.
        for (int s0 = 0; s0 < Sb; s0 += blockDim.x) {
            const int s = s0 + tid;
            uint32_t bin = 0xffffffffu, n = 0;
            if (s < Sb) {
                const uint32_t k = ordered_key(sc[s]);
                if ((k & mask) == prefix) {
                    bin = (k >> shift) & dmask;
                    n = (uint32_t)(o[s + 1] - o[s]);
                }
            }
            const uint32_t peers = __match_any_sync(0xffffffffu, bin);
            if (bin != 0xffffffffu) {
                const uint32_t wsum = __reduce_add_sync(peers, n);
                if ((tid & 31) == __ffs(peers) - 1) {
                    atomicAdd(&hw[bin], wsum);
                    atomicAdd(&hc[bin], (uint32_t)__popc(peers));
                }
            }
        }
        __syncthreads();
        // thread t owns bins 2t (lower) and 2t+1 (upper); weight above t's pair = total - incl
        const uint32_t w_lo = hw[2 * tid], w_hi = hw[2 * tid + 1];
        uint32_t total;
        const uint32_t incl = block_incl_sum<uint32_t>(w_lo + w_hi, ws32, &total);
        if (tid == 0) sh_found = 0;
        __syncthreads();
        if (pass == 0 && total <= rem) {
            all_fit = true;  // every sentence fits the budget
            break;
        }
        const uint32_t above = total - incl;  // weight of all bins above this pair
        if (above <= rem && above + w_hi > rem) {
            sh_bin = 2 * tid + 1;
            sh_rem = rem - above;
            sh_cnt = hc[2 * tid + 1];
            sh_found = 1;
        } else if (above + w_hi <= rem && above + w_hi + w_lo > rem) {
            sh_bin = 2 * tid;
            sh_rem = rem - above - w_hi;
            sh_cnt = hc[2 * tid];
            sh_found = 1;
        }
        __syncthreads();
        prefix |= sh_bin << shift;
        mask |= dmask << shift;
        rem = sh_rem;
        // A bin holding a single sentence: that sentence is s*; everything above is selected.
        if (sh_cnt == 1u) resolved = true;
        __syncthreads();
    }
    // Sentences with (key & mask) > prefix rank above the crossing range and are selected.
    // Inside the range (key & mask) == prefix: if resolved, the range is {s*} (not selected);
    // otherwise the range is a set of exact ties -> in index order, select while the cumulative
    // tied length stays <= rem.
    const bool ties = !all_fit && !resolved;

    uint32_t tie_carry = 0;
    unsigned long long carry = 0;  // (count << 32) | tokens of selected sentences so far
    int32_t* ids = sel_ids + (size_t)(b * G + g) * tau;
    int32_t* tokoff = sel_tokoff + (size_t)(b * G + g) * (tau + 1);
    for (int base = 0; base < Sb; base += blockDim.x) {
        const int s = base + tid;
        const bool valid = s < Sb;
        uint32_t k = 0, n = 0;
        if (valid) {
            k = ordered_key(sc[s]);
            n = (uint32_t)(o[s + 1] - o[s]);
        }
        bool sel;
        if (all_fit) {
            sel = valid;
        } else {
            const uint32_t km = k & mask;
            sel = valid && km > prefix;
            if (ties) {
                const uint32_t tw = (valid && km == prefix) ? n : 0u;
                uint32_t ttot;
                const uint32_t tincl = block_incl_sum<uint32_t>(tw, ws32, &ttot) + tie_carry;
                tie_carry += ttot;
                if (tw > 0u && tincl <= rem) sel = true;
            }
        }
        const unsigned long long v = sel ? ((1ull << 32) | (unsigned long long)n) : 0ull;
        unsigned long long vtot;
        const unsigned long long incl = block_incl_sum<unsigned long long>(v, ws64, &vtot) + carry;
        if (sel) {
            const unsigned long long excl = incl - v;
            const int pos = (int)(excl >> 32);
            ids[pos] = s;
            tokoff[pos] = (int32_t)(excl & 0xffffffffull);
        }
        carry += vtot;
    }
    const int count = (int)(carry >> 32);
    const int ntok = (int)(carry & 0xffffffffull);
    if (tid == 0) {
        tokoff[count] = ntok;
        sel_count[b * G + g] = count;
        if (out_count) out_count[b * G + g] = count;
        if (out_tokens) out_tokens[b * G + g] = ntok;
    }
    if (out_ids) {
        __syncthreads();
        int32_t* oi = out_ids + (size_t)(b * G + g) * tau;
        for (int i = tid; i < tau; i += blockDim.x) oi[i] = i < count ? ids[i] : -1;
    }
}

cudaError_t launch_select(const float* scores, const int32_t* off, int off_stride, const int32_t* S, int B,
                          int G, int grp, int d, int Smax, int tau, const __nv_bfloat16* q,
                          const int32_t* input_token, const int32_t* bset, int nb, float* Sq, int32_t* cnt,
                          int32_t* sel_ids, int32_t* sel_tokoff, int32_t* sel_count, int32_t* out_ids,
                          int32_t* out_count, int32_t* out_tokens, cudaStream_t st) {
    dim3 grid(G, B);
    select_kernel<<<grid, kSelThreads, 0, st>>>(scores, off, off_stride, S, G, grp, d, Smax, tau, q, input_token,
                                                bset, nb, Sq, cnt, sel_ids, sel_tokoff, sel_count, out_ids,
                                                out_count, out_tokens);
    return cudaGetLastError();
}

}  // namespace skv
