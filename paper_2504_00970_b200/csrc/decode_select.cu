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

SKV_TRACE_DEFINE(select)

// ------------------------------------------------------------------------------ D1 scoring
//
// Grid (splits, G, B); each CTA scores a contiguous range of sentences of one (b, g) unit.  The
// range's embeddings are contiguous in HBM ([B][G][Smax][d]), so they stream into shared memory
// as 16 KB tiles by single bulk async copies (TMA engine) through a kScStages-deep mbarrier
// pipeline; the first tiles are in flight while the CTA forms the group query
// qt_g = sum_h qbar_h, qbar_h = (Sq_h + q_h) / (cnt + 1) (the appended, not yet stored, Q_s of
// this step; the state itself is written by the select kernel, which runs after all scoring
// CTAs).  D/8 lanes per sentence: lane l holds qt[8l..8l+7] in registers and reads one 16-byte
// chunk of the sentence row from shared memory (conflict-free); the fp32 dot follows the
// canonical order (mul, 7 fma, then xor-butterfly adds whose lane-0 result equals the tree of
// A23).  E is read exactly once per step: the HBM-bound part of decode.
constexpr int kScThreads = 256;
constexpr int kScTileBytes = 16384;
constexpr int kScStages = 4;

template <int D, int GRP>
__global__ void __launch_bounds__(kScThreads) score_kernel(const __nv_bfloat16* __restrict__ q,
                                                           const float* __restrict__ Sq,
                                                           const int32_t* __restrict__ cnt,
                                                           const __nv_bfloat16* __restrict__ E,
                                                           const int32_t* __restrict__ S, int G, int Smax,
                                                           int chunk, float* __restrict__ scores, int qmode) {
    constexpr int LPS = D / 8;                   // lanes per sentence
    constexpr int GPW = 32 / LPS;                // sentences per warp step
    constexpr int TS = kScTileBytes / (D * 2);   // sentences per tile (64 or 128)
    constexpr int NW = kScThreads / 32;
    static_assert(TS % (NW * GPW) == 0, "tile must split evenly over the warps");
    extern __shared__ __align__(128) unsigned char sc_smem[];
    __nv_bfloat16* tiles = reinterpret_cast<__nv_bfloat16*>(sc_smem);  // [kScStages][TS*D]
    __shared__ uint64_t bar[kScStages];
    __shared__ float qt[D];

    const int b = blockIdx.z, g = blockIdx.y;
    pdl_wait();
    const int Sb = S[b];
    const int s0 = blockIdx.x * chunk;
    if (s0 >= Sb) return;
    const int s1 = min(Sb, s0 + chunk);
    const int ntiles = (s1 - s0 + TS - 1) / TS;
    const int Hq = G * GRP;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const __nv_bfloat16* Eu = E + ((size_t)(b * G + g) * Smax) * D;
    SKV_TRACE_POINT(24);

    if (tid == 0) {
        for (int i = 0; i < kScStages; ++i) mbar_init(&bar[i], 1);
        for (int i = 0; i < kScStages && i < ntiles; ++i) {
            const int ts = s0 + i * TS, n = min(TS, s1 - ts);
            mbar_arrive_expect_tx(&bar[i], (uint32_t)(n * D * 2));
            bulk_g2s(tiles + (size_t)i * TS * D, Eu + (size_t)ts * D, (uint32_t)(n * D * 2), &bar[i]);
        }
    }
    // group query of this step (loads batched, canonical order: qbar_h by IEEE division, then
    // ascending-h fp32 sum)
    if (tid < D) {
        const float c = (float)(cnt[b * G + g] + 1);
        float sv[GRP], qv[GRP];
#pragma unroll
        for (int h = 0; h < GRP; ++h) {
            const size_t idx = ((size_t)b * Hq + g * GRP + h) * D + tid;
            sv[h] = Sq[idx];
            qv[h] = __bfloat162float(q[idx]);
        }
        // qmode 1 (NEXT-3, Sec. 6.2): rank by the current token's query, qbar_h = q_h
        float acc = qmode ? qv[0] : __fdiv_rn(__fadd_rn(sv[0], qv[0]), c);
#pragma unroll
        for (int h = 1; h < GRP; ++h) acc = __fadd_rn(acc, qmode ? qv[h] : __fdiv_rn(__fadd_rn(sv[h], qv[h]), c));
        qt[tid] = acc;
    }
    __syncthreads();
    const int l = lane % LPS, gw = lane / LPS;
    float qr[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) qr[i] = qt[8 * l + i];
    float* out = scores + (size_t)(b * G + g) * Smax;
    SKV_TRACE_POINT(25);

    for (int it = 0; it < ntiles; ++it) {
        const int st = it % kScStages;
        mbar_wait(&bar[st], (it / kScStages) & 1);
        if (it == 0) SKV_TRACE_POINT(26);
        const __nv_bfloat16* tile = tiles + (size_t)st * TS * D;
        const int ts = s0 + it * TS, n = min(TS, s1 - ts);
#pragma unroll
        for (int j = 0; j < TS / (NW * GPW); ++j) {
            const int r = (j * NW + warp) * GPW + gw;  // sentence row within the tile
            float f[8];
            unpack8(*reinterpret_cast<const uint4*>(tile + (size_t)r * D + 8 * l), f);
            float p = __fmul_rn(qr[0], f[0]);
#pragma unroll
            for (int i = 1; i < 8; ++i) p = __fmaf_rn(qr[i], f[i], p);
#pragma unroll
            for (int o = LPS / 2; o >= 1; o >>= 1) p = __fadd_rn(p, __shfl_xor_sync(0xffffffffu, p, o));
            if (l == 0 && r < n) out[ts + r] = p;
        }
        __syncthreads();  // stage st fully read
        if (it + 1 == ntiles) pdl_trigger();
        if (tid == 0 && it + kScStages < ntiles) {
            const int tn = s0 + (it + kScStages) * TS, nn = min(TS, s1 - tn);
            mbar_arrive_expect_tx(&bar[st], (uint32_t)(nn * D * 2));
            bulk_g2s(tiles + (size_t)st * TS * D, Eu + (size_t)tn * D, (uint32_t)(nn * D * 2), &bar[st]);
        }
    }
}

template <int D, int GRP>
static cudaError_t launch_score_t(dim3 grid, int chunk, cudaStream_t st, const __nv_bfloat16* q, const float* Sq,
                                  const int32_t* cnt, const __nv_bfloat16* E, const int32_t* S, int G, int Smax,
                                  float* scores, int qmode) {
    const size_t smem = (size_t)kScStages * kScTileBytes;
    cudaError_t e = ensure_smem((const void*)score_kernel<D, GRP>, smem);
    if (e != cudaSuccess) return e;
    return launch_pdl_if(false, score_kernel<D, GRP>, grid, dim3(kScThreads), smem, st, q, Sq, cnt, E, S, G, Smax, chunk,
                      scores, qmode);
}

cudaError_t launch_score(const __nv_bfloat16* q, const float* Sq, const int32_t* cnt, const __nv_bfloat16* E,
                         const int32_t* S, int B, int G, int grp, int d, int Smax, float* scores, int qmode,
                         cudaStream_t st) {
    // ~3 CTAs per SM: split each (b, g) unit's sentences into `splits` tile-aligned ranges.
    const int TS = kScTileBytes / (d * 2);
    const int units = B * G;
    int splits = (3 * kNumSMs + units - 1) / units;
    int chunk = (Smax + splits - 1) / splits;
    chunk = max(TS, (chunk + TS - 1) / TS * TS);
    splits = (Smax + chunk - 1) / chunk;
    dim3 grid(splits, G, B);
#define SKV_SC(DV, GV) return launch_score_t<DV, GV>(grid, chunk, st, q, Sq, cnt, E, S, G, Smax, scores, qmode)
    if (d == 128) {
        switch (grp) {
            case 1: SKV_SC(128, 1);
            case 2: SKV_SC(128, 2);
            case 4: SKV_SC(128, 4);
            case 8: SKV_SC(128, 8);
        }
    } else {
        switch (grp) {
            case 1: SKV_SC(64, 1);
            case 2: SKV_SC(64, 2);
            case 4: SKV_SC(64, 4);
            case 8: SKV_SC(64, 8);
        }
    }
#undef SKV_SC
    return cudaErrorInvalidValue;
}

// ----------------------------------------------------------------------------- D2 selection
//
// One CTA (1024 threads) per (b, g).  The selection is the maximal prefix of the ranking by
// key64 = (ordered(score) << 32) | (0xffffffff - index) whose token count fits tau (A13, A14):
// find the first sentence s* in rank order at which the cumulative length exceeds tau, then
// select every sentence with key64 > key64(s*) (all sentences if the total fits).
//
// s* is located by range refinement on the 32-bit ordered score key k:
//   level: histogram (2048 bins, length-weighted and counted) of the sentences whose key lies
//   in [lo, hi], bin = (k - lo) * 2048 / (hi - lo + 1) (monotone in k, so bins are key
//   intervals); one block scan finds the bin where the cumulative length from the top crosses
//   the remaining budget.  If that bin holds <= 1024 sentences they are ranked exactly by key64
//   (one thread per candidate) and s* is found; otherwise [lo, hi] shrinks to the bin's key
//   range and the level repeats (at most 3 times for 32-bit keys).  If lo == hi the remaining
//   sentences tie on the score and s* is found in ascending index order (the tie rule) by one
//   ordered block scan.
// The ordered-key space is roughly logarithmic in the score, so bins are ~1/8 octave wide and
// the histogram atomics see little contention.  A final ordered block scan compacts the selected
// ids in ascending order with their token prefix sums.  Thread t owns the contiguous index range
// [t*E, t*E+E); keys and lengths are cached in shared memory (S <= kSelSmemCap).
//
// The deferred D1 state update (Sq += q_t, or reset at a boundary, A11) is done afterwards by the
// attend kernel (qs_update_unit), off the selection's critical path.
constexpr int kSelThreads = 1024;
constexpr int kBins = 2048;
constexpr int kSelSmemCap = 19000;  // 10 B per sentence of dynamic shared memory
constexpr int kCandCap = kSelThreads;

__device__ __forceinline__ unsigned long long key64_of(uint32_t k, int s) {
    return ((unsigned long long)k << 32) | (unsigned long long)(0xffffffffu - (uint32_t)s);
}

template <bool SMEM>
__global__ void __launch_bounds__(kSelThreads) select_kernel(
    const float* __restrict__ scores, const int32_t* __restrict__ off, int off_stride,
    const int32_t* __restrict__ S, int G, int Smax, int tau, SelBufs sel, bool src_gathered,
    int32_t* __restrict__ out_ids, int32_t* __restrict__ out_count, int32_t* __restrict__ out_tokens,
    const int32_t* __restrict__ sid, int sid_stride) {
    __shared__ uint32_t hist[kBins];  // length-weighted histogram
    __shared__ unsigned long long cand_key[kCandCap];
    __shared__ uint32_t cand_len[kCandCap];
    __shared__ uint32_t ws32[32];
    __shared__ unsigned long long ws64[32];
    __shared__ uint32_t sh_bin, sh_rem, sh_lo, sh_hi, sh_ncand;
    __shared__ unsigned long long sh_thr;
    extern __shared__ __align__(16) unsigned char sel_smem[];
    uint32_t* skey = reinterpret_cast<uint32_t*>(sel_smem);                    // [Smax] ordered keys
    int32_t* soff = reinterpret_cast<int32_t*>(sel_smem + 4 * (size_t)Smax);   // [Smax] first token
    uint16_t* slen = reinterpret_cast<uint16_t*>(sel_smem + 8 * (size_t)Smax);  // [Smax] (len <= tau <= 65535)

    const int g = blockIdx.x, b = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31;
    pdl_wait();
    const int Sb = S[b];
    const float* sc = scores + (size_t)(b * G + g) * Smax;
    const int32_t* o = off + (size_t)b * off_stride;

    SKV_TRACE_POINT(0);
    if (tid == 0) {
        sh_lo = 0xffffffffu;
        sh_hi = 0u;
        sh_ncand = 0u;
    }
    __syncthreads();
    // ---- keys, lengths and offsets -> shared memory (one batched pass) + the key range ----
    {
        uint32_t mn = 0xffffffffu, mx = 0u;
        constexpr int U = 8;
        for (int s0 = 0; s0 < Sb; s0 += U * kSelThreads) {
            float v[U];
            int a0[U], a1[U];
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const int s = s0 + j * kSelThreads + tid;
                v[j] = s < Sb ? sc[s] : 0.0f;
                a0[j] = s < Sb ? o[s] : 0;
                a1[j] = s < Sb ? o[s + 1] : 0;
            }
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const int s = s0 + j * kSelThreads + tid;
                if (s < Sb) {
                    const uint32_t k = ordered_key(v[j]);
                    mn = min(mn, k);
                    mx = max(mx, k);
                    if (SMEM) {
                        skey[s] = k;
                        soff[s] = a0[j];
                        slen[s] = (uint16_t)(a1[j] - a0[j]);
                    }
                }
            }
        }
        mn = __reduce_min_sync(0xffffffffu, mn);
        mx = __reduce_max_sync(0xffffffffu, mx);
        if (lane == 0) {
            atomicMin(&sh_lo, mn);
            atomicMax(&sh_hi, mx);
        }
    }
    __syncthreads();
    SKV_TRACE_POINT(2);
    auto key_of = [&](int s) -> uint32_t { return SMEM ? skey[s] : ordered_key(sc[s]); };
    auto len_of = [&](int s) -> uint32_t { return SMEM ? (uint32_t)slen[s] : (uint32_t)(o[s + 1] - o[s]); };
    auto off_of = [&](int s) -> int32_t { return SMEM ? soff[s] : o[s]; };
    const int E = (Sb + kSelThreads - 1) / kSelThreads;
    const int i0 = min(Sb, tid * E), i1 = min(Sb, i0 + E);
    SKV_TRACE_POINT(3);
    uint32_t lo = sh_lo, hi = sh_hi, rem = (uint32_t)tau;
    bool all_fit = false;
    unsigned long long thr = 0;  // select key64 > thr
    for (int level = 0;; ++level) {
        if (lo == hi) {
            // the remaining candidates all carry key lo: index order decides (tie rule)
            uint32_t tw = 0;
            for (int s = i0; s < i1; ++s)
                if (key_of(s) == lo) tw += len_of(s);
            uint32_t ttot;
            const uint32_t before = block_incl_sum<uint32_t>(tw, ws32, &ttot) - tw;
            if (level == 0 && ttot <= rem) {
                all_fit = true;
                break;
            }
            if (before <= rem && before + tw > rem) {
                uint32_t acc = before;
                for (int s = i0; s < i1; ++s) {
                    if (key_of(s) != lo) continue;
                    acc += len_of(s);
                    if (acc > rem) {
                        sh_thr = key64_of(lo, s);
                        break;
                    }
                }
            }
            __syncthreads();
            thr = sh_thr;
            break;
        }
        // bin(k) = (k - lo) * kBins / span, as a 32.32 fixed-point multiply (monotone in k, < kBins);
        // spans below kBins map one key per bin.
        const unsigned long long span = (unsigned long long)(hi - lo) + 1ull;
        const unsigned long long mul = span >= kBins ? ((unsigned long long)kBins << 32) / span : 0ull;
        auto bin_of = [&](uint32_t k) -> uint32_t {
            return mul ? (uint32_t)(((unsigned long long)(k - lo) * mul) >> 32) : (k - lo);
        };
        for (int i = tid; i < kBins; i += blockDim.x) hist[i] = 0u;
        __syncthreads();
        for (int s = i0; s < i1; ++s) {
            const uint32_t k = key_of(s);
            if (k < lo || k > hi) continue;
            atomicAdd(&hist[bin_of(k)], len_of(s));
        }
        __syncthreads();
        SKV_TRACE_POINT(4 + 4 * level);
        // thread t owns bins 2t (lower) and 2t+1 (upper); weight above t's pair = total - incl
        const uint32_t w_lo = hist[2 * tid], w_hi = hist[2 * tid + 1];
        uint32_t total;
        const uint32_t incl = block_incl_sum<uint32_t>(w_lo + w_hi, ws32, &total);
        if (level == 0 && total <= rem) {
            all_fit = true;
            break;
        }
        const uint32_t above = total - incl;
        if (above <= rem && above + w_hi > rem) {
            sh_bin = 2 * tid + 1;
            sh_rem = rem - above;
        } else if (above + w_hi <= rem && above + w_hi + w_lo > rem) {
            sh_bin = 2 * tid;
            sh_rem = rem - above - w_hi;
        }
        if (tid == 0) {
            sh_lo = 0xffffffffu;
            sh_hi = 0u;
            sh_ncand = 0u;
        }
        __syncthreads();
        SKV_TRACE_POINT(5 + 4 * level);
        const uint32_t cb = sh_bin;
        rem = sh_rem;
        // gather the crossing bin's sentences (at most kCandCap) and its key range in one pass
        {
            uint32_t mn = 0xffffffffu, mx = 0u;
            for (int s = i0; s < i1; ++s) {
                const uint32_t k = key_of(s);
                if (k < lo || k > hi || bin_of(k) != cb) continue;
                mn = min(mn, k);
                mx = max(mx, k);
                const uint32_t pos = atomicAdd(&sh_ncand, 1u);
                if (pos < (uint32_t)kCandCap) {
                    cand_key[pos] = key64_of(k, s);
                    cand_len[pos] = len_of(s);
                }
            }
            mn = __reduce_min_sync(0xffffffffu, mn);
            mx = __reduce_max_sync(0xffffffffu, mx);
            if (lane == 0) {
                atomicMin(&sh_lo, mn);
                atomicMax(&sh_hi, mx);
            }
        }
        __syncthreads();
        SKV_TRACE_POINT(6 + 4 * level);
        if (sh_ncand <= (uint32_t)kCandCap) {
            // exact rank of the crossing bin's sentences by key64
            const int nc = (int)sh_ncand;
            if (tid < nc) {
                const unsigned long long mk = cand_key[tid];
                uint32_t wabove = 0;
                for (int c = 0; c < nc; ++c)
                    if (cand_key[c] > mk) wabove += cand_len[c];
                if (wabove <= rem && wabove + cand_len[tid] > rem) sh_thr = mk;
            }
            __syncthreads();
            SKV_TRACE_POINT(7 + 4 * level);
            thr = sh_thr;
            break;
        }
        // too many candidates: narrow [lo, hi] to the crossing bin's key range and repeat
        lo = sh_lo;
        hi = sh_hi;
        __syncthreads();
    }
    pdl_trigger();
    // ---- ordered compaction of the selected sentences (ascending ids + token offsets) ----
    unsigned long long mine = 0;
    for (int s = i0; s < i1; ++s)
        if (all_fit || key64_of(key_of(s), s) > thr) mine += (1ull << 32) | len_of(s);
    unsigned long long tot;
    SKV_TRACE_POINT(20);
    const unsigned long long excl = block_incl_sum<unsigned long long>(mine, ws64, &tot) - mine;
    SKV_TRACE_POINT(21);
    // this step's selection goes to slot parity^1 (the previous one stays readable in slot parity)
    const int cur = sel.parity[b * G + g] ^ 1;
    int32_t* ids = sel.ids_of(cur, b * G + g);
    int32_t* tokoff = sel.tok_of(cur, b * G + g);
    int32_t* src = sel.src_of(cur, b * G + g);
    if (mine) {
        int pos = (int)(excl >> 32);
        uint32_t toff = (uint32_t)(excl & 0xffffffffull);
        for (int s = i0; s < i1; ++s) {
            if (all_fit || key64_of(key_of(s), s) > thr) {
                ids[pos] = s;
                tokoff[pos] = (int32_t)toff;
                src[pos] = src_gathered ? (int32_t)toff : off_of(s);
                if (out_ids) out_ids[(size_t)(b * G + g) * tau + pos] = sid ? sid[(size_t)b * sid_stride + s] : s;
                ++pos;
                toff += len_of(s);
            }
        }
    }
    const int count = (int)(tot >> 32);
    const int ntok = (int)(tot & 0xffffffffull);
    if (tid == 0) {
        tokoff[count] = ntok;
        *sel.count_of(cur, b * G + g) = count;
        if (out_count) out_count[b * G + g] = count;
        if (out_tokens) out_tokens[b * G + g] = ntok;
    }
    SKV_TRACE_POINT(22);
    if (out_ids)
        for (int i = count + tid; i < tau; i += blockDim.x) out_ids[(size_t)(b * G + g) * tau + i] = -1;
}

cudaError_t launch_select(const float* scores, const int32_t* off, int off_stride, const int32_t* S, int B,
                          int G, int Smax, int tau, SelBufs sel, bool src_gathered, int32_t* out_ids,
                          int32_t* out_count, int32_t* out_tokens, const int32_t* sid, int sid_stride,
                          cudaStream_t st) {
    dim3 grid(G, B);
    if (Smax <= kSelSmemCap && tau <= 65535) {
        const size_t smem = (size_t)Smax * 10 + 16;
        cudaError_t e = ensure_smem((const void*)select_kernel<true>, (size_t)(kSelSmemCap * 10 + 16));
        if (e != cudaSuccess) return e;
        return launch_pdl_if(false, select_kernel<true>, grid, dim3(kSelThreads), smem, st, scores, off, off_stride, S, G, Smax,
                          tau, sel, src_gathered, out_ids, out_count, out_tokens, sid, sid_stride);
    }
    return launch_pdl_if(false, select_kernel<false>, grid, dim3(kSelThreads), 0, st, scores, off, off_stride, S, G, Smax, tau,
                      sel, src_gathered, out_ids, out_count, out_tokens, sid, sid_stride);
}

}  // namespace skv
