// decode_layer.cu -- one persistent kernel per layer and decode step running D1 + D2 + D3 + D4 for
// every (b, g) unit of the context (device residency).
//
// Same arithmetic and results as score_kernel + select_kernel + attend_mma_kernel; this file only
// changes the schedule.  Those three kernels run back to back per layer, each paying its launch,
// ramp-up and drain, and HBM idles while the latency-bound selection runs.  Here the GPU is
// filled once with persistent CTAs (2 per SM) that take work items from a queue (one atomic
// ticket) in an order fixed per prompt on the host:
//   SCORE(u, k)  -- D1 for sentences [k*kLScore, ...) of unit u (TMA-streamed E, canonical dot);
//   SELECT(u)    -- D2 for unit u (+ the deferred Eq. 2 state update); waits for u's SCOREs;
//   ATTEND(u, c) -- D3 + D4 for gathered tokens [c*kLAtt, ...) of u (mma.sync tiles); waits for
//                   SELECT(u); the last ATTEND of u merges the partials and writes O.
// Units are interleaved in groups (score group k, then select group k-1, then attend group k-2...),
// so one group's selection runs while other groups stream E or K/V from HBM.  An item only waits
// on items placed earlier in the queue, which are already held by resident CTAs, so the waits
// cannot deadlock.  Dependencies are per-unit counters in global memory (release: fence + atomic;
// acquire: ld.acquire + fence); produced data is read with L1-bypassing loads.
#include <algorithm>
#include <cstdlib>
#include <cstddef>
#include <vector>

#include "device_util.cuh"
#include "skv_internal.cuh"

namespace skv {
SKV_TRACE_DEFINE(layer)
#ifdef SKV_TRACE
// per work item: globaltimer at claim and at completion (ns; comparable across SMs)
__device__ unsigned long long g_item_t[2048][2];
extern "C" __attribute__((visibility("default"))) int sentencekv_debug_items(unsigned long long* out, int n) {
    return (int)cudaMemcpyFromSymbol(out, g_item_t, sizeof(unsigned long long) * 2 * (size_t)n);
}
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ unsigned long long g_phase_t[64][16];  // [unit][phase] of SELECT items
extern "C" __attribute__((visibility("default"))) int sentencekv_debug_phases(unsigned long long* out) {
    return (int)cudaMemcpyFromSymbol(out, g_phase_t, sizeof(g_phase_t));
}
#define SKV_PHASE(u, ph)                                             \
    do {                                                             \
        if (threadIdx.x == 0 && (u) < 64) g_phase_t[(u)][(ph)] = gtime(); \
    } while (0)
#else
#define SKV_PHASE(u, ph) \
    do {                 \
    } while (0)
#endif

namespace {

constexpr int kLT = 256;                  // threads per CTA
constexpr int kLW = kLT / 32;
constexpr int kLScoreTiles = 8;           // 16 KB E tiles per SCORE item
constexpr int kLTileBytes = 16384;
constexpr int kLStages = 4;
constexpr int kLAtt = 256;                // gathered tokens per ATTEND item
constexpr int kTileT = 16;                // tokens per mma tile
constexpr int kLBins = 2048;
constexpr int kLCand = 1024;
constexpr int kInvalidRow = INT32_MIN;

enum : int { kItemScore = 0, kItemSelect = 1, kItemAttend = 2 };

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// thread 0 waits until *flag >= target, then the CTA may read what the producers released
__device__ __forceinline__ void cta_wait(const uint32_t* flag, uint32_t target) {
    if (threadIdx.x == 0)
        while (ld_acquire(flag) < target) __nanosleep(64);
    __syncthreads();
    __threadfence();
}

// all threads' writes become visible before the counter moves
__device__ __forceinline__ void cta_release(uint32_t* flag) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(flag, 1u);
}

__device__ __forceinline__ int ldcg_i(const int32_t* p) { return __ldcg(p); }

__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t w_of(const uint4& v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }
__device__ __forceinline__ uint32_t pair_elem(const uint4& x, const uint4& y, int e) {
    return __byte_perm(w_of(x, e >> 1), w_of(y, e >> 1), (e & 1) ? 0x7632 : 0x5410);
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(lo)) |
           ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(hi)) << 16);
}
__device__ __forceinline__ uint4 ldg16(const __nv_bfloat16* p) { return *reinterpret_cast<const uint4*>(p); }
__device__ __forceinline__ unsigned long long k64(uint32_t k, int s) {
    return ((unsigned long long)k << 32) | (unsigned long long)(0xffffffffu - (uint32_t)s);
}

// Shared memory of one persistent CTA; the item kinds use it one at a time.  Layout: control
// fields, then a union of the per-kind buffers, then (from tail_offset()) a tail sized at launch:
// SELECT's key/length cache (S_max x 6 B) or ATTEND's copy of the selection (2 tau + 1 ints).
template <int D>
struct LayerSmem {
    unsigned long long ws64[32];
    uint32_t ws32[32];
    uint32_t lo, hi, cb, rem, ncb, ncand, red_lo, red_hi;
    unsigned long long thr;
    int item;
    int last;
    union U {
        struct {
            alignas(128) __nv_bfloat16 tiles[kLStages][kLTileBytes / 2];
            uint64_t bar[kLStages];
            float qt[D];
            unsigned long long ukey[kLScoreTiles * kLTileBytes / (2 * D)];  // item's keys, index order
            unsigned long long skey[kLT / 2];                                 // local histogram scratch
        } sc;
        struct {
            unsigned long long hist[kLBins];
            unsigned long long cand_key[kLCand];
            uint32_t cand_len[kLCand];
        } se;
        struct {
            float red[kLW][8][D];
            float mw[kLW][8], lw[kLW][8];
            int32_t rowtab[kLAtt];
        } at;
    } u;
    __host__ __device__ static constexpr size_t tail_offset() {
        return (offsetof(LayerSmem, u) + (sizeof(U::se) > sizeof(U::at) ? sizeof(U::se) : sizeof(U::at)) + 15) / 16 * 16;
    }
    __device__ unsigned char* tail() { return reinterpret_cast<unsigned char*>(this) + tail_offset(); }
};

}  // namespace


// ------------------------------------------------------------------ D2, part 1 (inside D1 items)
// Local candidates of one SCORE item's sentence range [s0, s1): every sentence whose score lies in
// or above the item's local crossing bin -- a 256-bin length-weighted histogram of the item's
// keys, scanned from the top until the cumulative length exceeds tau.  This is a superset of the
// item's maximal prefix by key64 = (ordered score, -index) with lengths fitting tau plus the first
// sentence that does not fit; every sentence of the unit's selection, and the unit's crossing
// sentence, is therefore among the candidates of its item (the sentences ranked above it locally
// are a subset of those ranked above it globally), so SELECT only has to rank the candidates.
// Written in ascending index order, so the unit's lists concatenate in ascending sentence order.
template <int D>
__device__ void local_candidates(const LayerArgs& a, LayerSmem<D>& sm, int u, int k, int s0, int s1) {
    constexpr int NL = kLScoreTiles * kLTileBytes / (2 * D);  // 512 (D=128) or 1024 (D=64)
    constexpr int NB = kLT;                                   // local bins
    constexpr int E = NL / kLT;
    const int tid = threadIdx.x, lane = tid & 31;
    const int b = u / a.G;
    const int n = s1 - s0;
    const int32_t* o = a.off + (size_t)b * a.off_stride;
    uint32_t* hist = reinterpret_cast<uint32_t*>(sm.u.sc.skey);  // [NB] (skey is free scratch here)
    uint32_t key[E], len[E];
    uint32_t mn = 0xffffffffu, mx = 0u;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = E * tid + e;
        key[e] = i < n ? (uint32_t)(sm.u.sc.ukey[i] >> 32) : 0u;
        len[e] = i < n ? (uint32_t)(o[s0 + i + 1] - o[s0 + i]) : 0u;
        if (i < n) {
            mn = min(mn, key[e]);
            mx = max(mx, key[e]);
        }
    }
    mn = __reduce_min_sync(0xffffffffu, mn);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (tid == 0) {
        sm.lo = 0xffffffffu;
        sm.hi = 0u;
    }
    hist[tid] = 0u;
    __syncthreads();
    if (lane == 0 && mx >= mn) {
        atomicMin(&sm.lo, mn);
        atomicMax(&sm.hi, mx);
    }
    __syncthreads();
    const uint32_t lo = sm.lo, hi = sm.hi;
    const unsigned long long span = (unsigned long long)(hi - lo) + 1ull;
    const unsigned long long mul = span >= NB ? ((unsigned long long)NB << 32) / span : 0ull;
    auto bin_of = [&](uint32_t kk) -> uint32_t {
        return mul ? (uint32_t)(((unsigned long long)(kk - lo) * mul) >> 32) : (kk - lo);
    };
#pragma unroll
    for (int e = 0; e < E; ++e)
        if (E * tid + e < n) atomicAdd(&hist[bin_of(key[e])], len[e]);
    __syncthreads();
    // thread t <-> bin NB-1-t: cumulative weight from the top
    const uint32_t w = hist[NB - 1 - tid];
    uint32_t tot;
    const uint32_t incl = block_incl_sum<uint32_t>(w, sm.ws32, &tot);
    if (tid == 0) sm.cb = 0u;  // everything fits: all sentences are candidates
    __syncthreads();
    if (incl - w <= (uint32_t)a.tau && incl > (uint32_t)a.tau) sm.cb = (uint32_t)(NB - 1 - tid);
    __syncthreads();
    const uint32_t cb = sm.cb;
    uint32_t cnt = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) cnt += (E * tid + e < n && bin_of(key[e]) >= cb) ? 1u : 0u;
    uint32_t ctot;
    uint32_t pos = block_incl_sum<uint32_t>(cnt, sm.ws32, &ctot) - cnt;
    int4* cand = a.cand + ((size_t)u * a.n_score_max + k) * NL;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = E * tid + e;
        if (i < n && bin_of(key[e]) >= cb) cand[pos++] = make_int4(s0 + i, (int)key[e], (int)len[e], 0);
    }
    if (tid == 0) a.cand_count[u * a.n_score_max + k] = (int)ctot;
}

// ------------------------------------------------------------------------------------------ D1
template <int D, int GRP>
__device__ void score_item(const LayerArgs& a, LayerSmem<D>& sm, int u, int k) {
    constexpr int LPS = D / 8, GPW = 32 / LPS, TS = kLTileBytes / (D * 2);
    const int b = u / a.G, g = u % a.G;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int Sb = a.S[b];
    const int s0 = k * kLScoreTiles * TS;
    const int s1 = min(Sb, s0 + kLScoreTiles * TS);
    const int ntiles = s0 < s1 ? (s1 - s0 + TS - 1) / TS : 0;
    const __nv_bfloat16* Eu = a.E + (size_t)u * a.Smax * D;
    if (tid == 0) {
        for (int i = 0; i < kLStages; ++i) mbar_init(&sm.u.sc.bar[i], 1);
        for (int i = 0; i < kLStages && i < ntiles; ++i) {
            const int ts = s0 + i * TS, n = min(TS, s1 - ts);
            mbar_arrive_expect_tx(&sm.u.sc.bar[i], (uint32_t)(n * D * 2));
            bulk_g2s(sm.u.sc.tiles[i], Eu + (size_t)ts * D, (uint32_t)(n * D * 2), &sm.u.sc.bar[i]);
        }
    }
    const int Hq = a.G * GRP;
    if (tid < D) {  // group query of this step, canonical order (A23)
        const float c = (float)(a.cnt[u] + 1);
        float sv[GRP], qv[GRP];
#pragma unroll
        for (int h = 0; h < GRP; ++h) {
            const size_t idx = ((size_t)b * Hq + g * GRP + h) * D + tid;
            sv[h] = a.Sq[idx];
            qv[h] = __bfloat162float(a.q[idx]);
        }
        float acc = __fdiv_rn(__fadd_rn(sv[0], qv[0]), c);
#pragma unroll
        for (int h = 1; h < GRP; ++h) acc = __fadd_rn(acc, __fdiv_rn(__fadd_rn(sv[h], qv[h]), c));
        sm.u.sc.qt[tid] = acc;
    }
    __syncthreads();
    const int l = lane % LPS, gw = lane / LPS;
    float qr[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) qr[i] = sm.u.sc.qt[8 * l + i];
    float* outp = a.scores + (size_t)u * a.Smax;
    for (int it = 0; it < ntiles; ++it) {
        const int st = it % kLStages;
        mbar_wait(&sm.u.sc.bar[st], (it / kLStages) & 1);
        const __nv_bfloat16* tile = sm.u.sc.tiles[st];
        const int ts = s0 + it * TS, n = min(TS, s1 - ts);
#pragma unroll
        for (int j = 0; j < TS / (kLW * GPW); ++j) {
            const int r = (j * kLW + warp) * GPW + gw;
            float f[8];
            unpack8(*reinterpret_cast<const uint4*>(tile + (size_t)r * D + 8 * l), f);
            float p = __fmul_rn(qr[0], f[0]);
#pragma unroll
            for (int i = 1; i < 8; ++i) p = __fmaf_rn(qr[i], f[i], p);
#pragma unroll
            for (int o = LPS / 2; o >= 1; o >>= 1) p = __fadd_rn(p, __shfl_xor_sync(0xffffffffu, p, o));
            if (l == 0 && r < n) {
                outp[ts + r] = p;
                sm.u.sc.ukey[ts + r - s0] = k64(ordered_key(p), ts + r);
            }
        }
        __syncthreads();
        if (tid == 0 && it + kLStages < ntiles) {
            const int tn = s0 + (it + kLStages) * TS, nn = min(TS, s1 - tn);
            mbar_arrive_expect_tx(&sm.u.sc.bar[st], (uint32_t)(nn * D * 2));
            bulk_g2s(sm.u.sc.tiles[st], Eu + (size_t)tn * D, (uint32_t)(nn * D * 2), &sm.u.sc.bar[st]);
        }
    }
    if (tid == 0)
        for (int i = 0; i < kLStages; ++i)
            asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_addr(&sm.u.sc.bar[i])) : "memory");
    local_candidates<D>(a, sm, u, k, s0, s1);
    cta_release(&a.score_done[u]);
}

// ------------------------------------------------------------------------------------------ D2
// The selection of select_kernel (decode_select.cu) for one unit on kLT threads, run over the
// unit's candidates (local_candidates, in ascending sentence order) instead of all S sentences:
// range-binned length-weighted histogram -> crossing bin -> exact rank of its entries (or a
// narrower range, or the tie rule) -> ordered compaction.
template <int D, int GRP>
__device__ void select_item(const LayerArgs& a, LayerSmem<D>& sm, int u, int n_score) {
    const int b = u / a.G, g = u % a.G;
    const int tid = threadIdx.x, lane = tid & 31;
    SKV_PHASE(u, 0);
    cta_wait(&a.score_done[u], (uint32_t)n_score);
    SKV_PHASE(u, 1);
    const int32_t* o = a.off + (size_t)b * a.off_stride;
    const int Hq = a.G * GRP;
    const int tau = a.tau;
    // deferred D1 state update of this unit's heads (Eq. 2 cache; reset at a boundary input, A11)
    {
        const bool reset = in_set(a.input_token[b], a.bset, a.nb);
        const size_t base = ((size_t)b * Hq + (size_t)g * GRP) * D;
        for (int i = tid; i < GRP * D; i += kLT)
            a.Sq[base + i] = reset ? 0.0f : __fadd_rn(a.Sq[base + i], __bfloat162float(a.q[base + i]));
        if (tid == 0) a.cnt[u] = reset ? 0 : a.cnt[u] + 1;
    }
    // gather the candidate lists of the unit's SCORE items (ascending sentence order)
    constexpr int NL = kLScoreTiles * kLTileBytes / (2 * D);
    int32_t* cbase = reinterpret_cast<int32_t*>(sm.tail());       // [n_score + 1] list offsets
    int32_t* cid = cbase + (a.n_score_max + 1);                   // [Smax] sentence ids
    uint32_t* skey = reinterpret_cast<uint32_t*>(cid + a.Smax);   // [Smax] ordered score keys
    uint32_t* slen = skey + a.Smax;                               // [Smax] lengths
    if (tid < 32) {  // list offsets: warp scan of the per-item candidate counts
        int acc = 0;
        for (int k0 = 0; k0 < n_score; k0 += 32) {
            const int k = k0 + tid;
            const int c = k < n_score ? ldcg_i(a.cand_count + u * a.n_score_max + k) : 0;
            const int incl = warp_incl_sum(c);
            if (k < n_score) cbase[k] = acc + incl - c;
            acc += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (tid == 0) cbase[n_score] = acc;
    }
    __syncthreads();
    const int Sb = cbase[n_score];  // candidates of the unit
    SKV_PHASE(u, 2);
    for (int j0 = 0; j0 < Sb; j0 += 4 * kLT) {  // flat, batched loads of all lists
        int4 v[4];
        int jj[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int j = j0 + r * kLT + tid;
            jj[r] = j;
            v[r] = make_int4(0, 0, 0, 0);
            if (j < Sb) {
                int lo = 0, hi = n_score - 1;  // list holding candidate j: largest k with cbase[k] <= j
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (cbase[mid] <= j) lo = mid; else hi = mid - 1;
                }
                v[r] = __ldcg(a.cand + ((size_t)u * a.n_score_max + lo) * NL + (j - cbase[lo]));
            }
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
            if (jj[r] < Sb) {
                cid[jj[r]] = v[r].x;
                skey[jj[r]] = (uint32_t)v[r].y;
                slen[jj[r]] = (uint32_t)v[r].z;
            }
    }
    __syncthreads();
    SKV_PHASE(u, 3);
    const int E = (Sb + kLT - 1) / kLT;
    const int i0 = min(Sb, tid * E), i1 = min(Sb, i0 + E);
    auto key_of = [&](int i) -> uint32_t { return skey[i]; };
    auto len_of = [&](int i) -> uint32_t { return slen[i]; };
    auto id_of = [&](int i) -> int { return cid[i]; };
    if (tid == 0) {
        sm.lo = 0xffffffffu;
        sm.hi = 0u;
    }
    __syncthreads();
    {
        uint32_t mn = 0xffffffffu, mx = 0u;
        for (int s = i0; s < i1; ++s) {
            const uint32_t k = key_of(s);
            mn = min(mn, k);
            mx = max(mx, k);
        }
        mn = __reduce_min_sync(0xffffffffu, mn);
        mx = __reduce_max_sync(0xffffffffu, mx);
        if (lane == 0) {
            atomicMin(&sm.lo, mn);
            atomicMax(&sm.hi, mx);
        }
    }
    __syncthreads();
    SKV_PHASE(u, 4);
    uint32_t lo = sm.lo, hi = sm.hi, rem = (uint32_t)tau;
    bool all_fit = false;
    unsigned long long thr = 0ull;
    for (int level = 0;; ++level) {
        if (lo == hi) {  // the remaining candidates tie on the score: index order decides
            uint32_t tw = 0;
            for (int s = i0; s < i1; ++s)
                if (key_of(s) == lo) tw += len_of(s);
            uint32_t ttot;
            const uint32_t before = block_incl_sum<uint32_t>(tw, sm.ws32, &ttot) - tw;
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
                        sm.thr = k64(lo, id_of(s));
                        break;
                    }
                }
            }
            __syncthreads();
            thr = sm.thr;
            break;
        }
        const unsigned long long span = (unsigned long long)(hi - lo) + 1ull;
        const unsigned long long mul = span >= kLBins ? ((unsigned long long)kLBins << 32) / span : 0ull;
        auto bin_of = [&](uint32_t k) -> uint32_t {
            return mul ? (uint32_t)(((unsigned long long)(k - lo) * mul) >> 32) : (k - lo);
        };
        for (int i = tid; i < kLBins; i += kLT) sm.u.se.hist[i] = 0ull;
        __syncthreads();
        for (int s = i0; s < i1; ++s) {
            const uint32_t k = key_of(s);
            if (k < lo || k > hi) continue;
            atomicAdd(&sm.u.se.hist[bin_of(k)], (1ull << 32) | len_of(s));
        }
        __syncthreads();
        // thread t owns bins [8t, 8t+8): weight above its group, then scan its bins from the top
        constexpr int BPT = kLBins / kLT;
        unsigned long long wsum = 0;
#pragma unroll
        for (int j = 0; j < BPT; ++j) wsum += sm.u.se.hist[BPT * tid + j] & 0xffffffffull;
        unsigned long long total;
        const unsigned long long incl = block_incl_sum<unsigned long long>(wsum, sm.ws64, &total);
        if (level == 0 && total <= rem) {
            all_fit = true;
            break;
        }
        unsigned long long above = total - incl;
        if (tid == 0) sm.ncand = 0u;
#pragma unroll
        for (int j = BPT - 1; j >= 0; --j) {
            const unsigned long long v = sm.u.se.hist[BPT * tid + j];
            const unsigned long long w = v & 0xffffffffull;
            if (above <= rem && above + w > rem) {
                sm.cb = (uint32_t)(BPT * tid + j);
                sm.rem = (uint32_t)(rem - above);
                sm.ncb = (uint32_t)(v >> 32);
            }
            above += w;
        }
        __syncthreads();
        const uint32_t cb = sm.cb, ncb = sm.ncb;
        rem = sm.rem;
        if (ncb <= (uint32_t)kLCand) {
            for (int s = i0; s < i1; ++s) {
                const uint32_t k = key_of(s);
                if (k < lo || k > hi || bin_of(k) != cb) continue;
                const uint32_t pos = atomicAdd(&sm.ncand, 1u);
                sm.u.se.cand_key[pos] = k64(k, id_of(s));
                sm.u.se.cand_len[pos] = len_of(s);
            }
            __syncthreads();
            const int nc = (int)sm.ncand;
            for (int c = tid; c < nc; c += kLT) {
                const unsigned long long mk = sm.u.se.cand_key[c];
                uint32_t wabove = 0;
                for (int j = 0; j < nc; ++j)
                    if (sm.u.se.cand_key[j] > mk) wabove += sm.u.se.cand_len[j];
                if (wabove <= rem && wabove + sm.u.se.cand_len[c] > rem) sm.thr = mk;
            }
            __syncthreads();
            thr = sm.thr;
            break;
        }
        {  // narrow [lo, hi] to the crossing bin's key range and repeat
            uint32_t mn = 0xffffffffu, mx = 0u;
            for (int s = i0; s < i1; ++s) {
                const uint32_t k = key_of(s);
                if (k < lo || k > hi || bin_of(k) != cb) continue;
                mn = min(mn, k);
                mx = max(mx, k);
            }
            mn = __reduce_min_sync(0xffffffffu, mn);
            mx = __reduce_max_sync(0xffffffffu, mx);
            if (tid == 0) {
                sm.red_lo = 0xffffffffu;
                sm.red_hi = 0u;
            }
            __syncthreads();
            if (lane == 0) {
                atomicMin(&sm.red_lo, mn);
                atomicMax(&sm.red_hi, mx);
            }
            __syncthreads();
            lo = sm.red_lo;
            hi = sm.red_hi;
        }
    }
    SKV_PHASE(u, 5);
    // ordered compaction into slot parity^1
    unsigned long long mine = 0;
    for (int s = i0; s < i1; ++s)
        if (all_fit || k64(key_of(s), id_of(s)) > thr) mine += (1ull << 32) | len_of(s);
    unsigned long long tot;
    const unsigned long long excl = block_incl_sum<unsigned long long>(mine, sm.ws64, &tot) - mine;
    const int cur = a.sel.parity[u] ^ 1;
    int32_t* ids = a.sel.ids_of(cur, u);
    int32_t* tokoff = a.sel.tok_of(cur, u);
    int32_t* src = a.sel.src_of(cur, u);
    if (mine) {
        int pos = (int)(excl >> 32);
        uint32_t toff = (uint32_t)(excl & 0xffffffffull);
        for (int s = i0; s < i1; ++s) {
            if (!(all_fit || k64(key_of(s), id_of(s)) > thr)) continue;
            const int sid = id_of(s);
            ids[pos] = sid;
            tokoff[pos] = (int32_t)toff;
            src[pos] = o[sid];  // context row of the sentence's first token
            if (a.out_ids) a.out_ids[(size_t)u * tau + pos] = sid;
            ++pos;
            toff += len_of(s);
        }
    }
    const int count = (int)(tot >> 32);
    if (tid == 0) {
        tokoff[count] = (int32_t)(tot & 0xffffffffull);
        *a.sel.count_of(cur, u) = count;
        if (a.out_count) a.out_count[u] = count;
        if (a.out_tokens) a.out_tokens[u] = (int32_t)(tot & 0xffffffffull);
    }
    if (a.out_ids)
        for (int i = count + tid; i < tau; i += kLT) a.out_ids[(size_t)u * tau + i] = -1;
    SKV_PHASE(u, 6);
    cta_release(&a.select_done[u]);
    SKV_PHASE(u, 7);
}

// --------------------------------------------------------------------------------------- D3+D4
// Gathered tokens [c*kLAtt, (c+1)*kLAtt) of unit u on tensor cores (attend_mma_kernel's tile
// math); the CTA partial (max, sum, unnormalised O) goes to the workspace; the last ATTEND of the
// unit merges the n_att partials and writes O.
template <int D, int GRP>
__device__ void attend_item(const LayerArgs& a, LayerSmem<D>& sm, int u, int c) {
    constexpr int NKS = D / 16, NU = D / 32, NVP = D / 64;
    const int b = u / a.G, g = u % a.G;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int gq = lane >> 2, cq = lane & 3;
    const int Hq = a.G * GRP;
    cta_wait(&a.select_done[u], 1u);
    const int cur = ldcg_i(a.sel.parity + u) ^ 1;
    const int count = ldcg_i(a.sel.count_of(cur, u));
    int32_t* tok = reinterpret_cast<int32_t*>(sm.tail());  // [count + 1]
    int32_t* srcs = tok + (a.tau + 1);                     // [count]
    {
        const int32_t* gt = a.sel.tok_of(cur, u);
        const int32_t* gs = a.sel.src_of(cur, u);
        for (int i = tid; i <= count; i += kLT) {
            tok[i] = ldcg_i(gt + i);
            if (i < count) srcs[i] = ldcg_i(gs + i);
        }
    }
    __syncthreads();
    const int ntok = tok[count];
    const int T0 = c * kLAtt, T1 = min(ntok, T0 + kLAtt);
    // row of every gathered token of this item
    for (int t = T0 + tid; t < T0 + kLAtt; t += kLT) {
        int r = kInvalidRow;
        if (t < T1) {
            int lo = 0, hi = count - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (tok[mid] <= t) lo = mid; else hi = mid - 1;
            }
            r = srcs[lo] + (t - tok[lo]);
        }
        sm.u.at.rowtab[t - T0] = r;
    }
    __syncthreads();
    const __nv_bfloat16* Kd = a.kv.K + (size_t)u * a.kv.unit_stride * D;
    const __nv_bfloat16* Vd = a.kv.V + (size_t)u * a.kv.unit_stride * D;
    uint4 qseg[NU];
#pragma unroll
    for (int uu = 0; uu < NU; ++uu)
        qseg[uu] = gq < GRP ? ldg16(a.q + ((size_t)b * Hq + g * GRP + gq) * D + (4 * uu + cq) * 8)
                            : make_uint4(0, 0, 0, 0);
    float m2[2] = {-INFINITY, -INFINITY}, l2[2] = {0.0f, 0.0f};
    float acc[NKS][4];
#pragma unroll
    for (int i = 0; i < NKS; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0f;
    const int ntile = T1 > T0 ? (T1 - T0 + kTileT - 1) / kTileT : 0;
    for (int tile = warp; tile < ntile; tile += kLW) {
        const int tl = tile * kTileT;  // local token offset
        const int rk0 = sm.u.at.rowtab[tl + gq], rk1 = sm.u.at.rowtab[tl + gq + 8];
        uint4 kA[NU], kB[NU];
#pragma unroll
        for (int uu = 0; uu < NU; ++uu) {
            kA[uu] = rk0 != kInvalidRow ? ldg16(Kd + (size_t)rk0 * D + (4 * uu + cq) * 8) : make_uint4(0, 0, 0, 0);
            kB[uu] = rk1 != kInvalidRow ? ldg16(Kd + (size_t)rk1 * D + (4 * uu + cq) * 8) : make_uint4(0, 0, 0, 0);
        }
        uint4 vv[4][NVP];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            const int rv = sm.u.at.rowtab[tl + 2 * cq + (kk & 1) + 8 * (kk >> 1)];
#pragma unroll
            for (int p = 0; p < NVP; ++p)
                vv[kk][p] = rv != kInvalidRow ? ldg16(Vd + (size_t)rv * D + 8 * gq + 64 * p) : make_uint4(0, 0, 0, 0);
        }
        float s[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int j = 0; j < NKS; ++j) {
            const int uu = j >> 1, h = (j & 1) * 2;
            const uint32_t af[4] = {w_of(kA[uu], h), w_of(kB[uu], h), w_of(kA[uu], h + 1), w_of(kB[uu], h + 1)};
            mma_bf16(s, af, w_of(qseg[uu], h), w_of(qseg[uu], h + 1));
        }
        const bool v0 = T0 + tl + gq < T1, v1 = T0 + tl + gq + 8 < T1;
        float p[4];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const bool hv = 2 * cq + e < GRP;
            const float sa = (hv && v0) ? s[e] * a.scale_log2 : -INFINITY;
            const float sb = (hv && v1) ? s[2 + e] * a.scale_log2 : -INFINITY;
            float mx = fmaxf(sa, sb);
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
            const float m_new = fmaxf(m2[e], mx);
            const float mref = m_new == -INFINITY ? 0.0f : m_new;
            p[e] = exp2f(sa - mref);
            p[2 + e] = exp2f(sb - mref);
            float sum = p[e] + p[2 + e];
            sum += __shfl_xor_sync(0xffffffffu, sum, 4);
            sum += __shfl_xor_sync(0xffffffffu, sum, 8);
            sum += __shfl_xor_sync(0xffffffffu, sum, 16);
            const float scl = exp2f(m2[e] - mref);
            l2[e] = l2[e] * scl + sum;
            m2[e] = m_new;
#pragma unroll
            for (int i = 0; i < NKS; ++i) {
                acc[i][e] *= scl;
                acc[i][2 + e] *= scl;
            }
        }
        const int X = 8 * cq + (gq >> 1), Y = X + 4, sel0 = gq & 1;
        float px[4], py[4];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            px[kk] = __shfl_sync(0xffffffffu, p[kk], X);
            py[kk] = __shfl_sync(0xffffffffu, p[kk], Y);
        }
        const float p00 = sel0 ? px[1] : px[0], p01 = sel0 ? py[1] : py[0];
        const float p10 = sel0 ? px[3] : px[2], p11 = sel0 ? py[3] : py[2];
        const uint32_t bh0 = pack_bf16(p00, p01), bh1 = pack_bf16(p10, p11);
        const uint32_t bl0 = pack_bf16(p00 - bf16lo(bh0), p01 - bf16hi(bh0));
        const uint32_t bl1 = pack_bf16(p10 - bf16lo(bh1), p11 - bf16hi(bh1));
#pragma unroll
        for (int i = 0; i < NKS; ++i) {
            uint32_t af[4];
            if (D == 128) {
                af[0] = pair_elem(vv[0][0], vv[1][0], i);
                af[1] = pair_elem(vv[0][NVP - 1], vv[1][NVP - 1], i);
                af[2] = pair_elem(vv[2][0], vv[3][0], i);
                af[3] = pair_elem(vv[2][NVP - 1], vv[3][NVP - 1], i);
            } else {
                af[0] = pair_elem(vv[0][0], vv[1][0], 2 * i);
                af[1] = pair_elem(vv[0][0], vv[1][0], 2 * i + 1);
                af[2] = pair_elem(vv[2][0], vv[3][0], 2 * i);
                af[3] = pair_elem(vv[2][0], vv[3][0], 2 * i + 1);
            }
            mma_bf16(acc[i], af, bh0, bh1);
            mma_bf16(acc[i], af, bl0, bl1);
        }
    }
    // ---- CTA partial: merge the warps ----
    if (gq == 0) {
        sm.u.at.mw[warp][2 * cq] = m2[0];
        sm.u.at.mw[warp][2 * cq + 1] = m2[1];
        sm.u.at.lw[warp][2 * cq] = l2[0];
        sm.u.at.lw[warp][2 * cq + 1] = l2[1];
    }
    __syncthreads();
    float wsc[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kLW; ++w) M = fmaxf(M, sm.u.at.mw[w][2 * cq + e]);
        wsc[e] = (m2[e] == -INFINITY) ? 0.0f : exp2f(m2[e] - M);
    }
#pragma unroll
    for (int i = 0; i < NKS; ++i)
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const int dim = (D == 128) ? (half ? 64 + 8 * gq + i : 8 * gq + i) : (8 * gq + 2 * i + half);
            sm.u.at.red[warp][2 * cq][dim] = acc[i][2 * half] * wsc[0];
            sm.u.at.red[warp][2 * cq + 1][dim] = acc[i][2 * half + 1] * wsc[1];
        }
    __syncthreads();
    float* pml = a.part_ml + ((size_t)u * a.n_att + c) * 16;
    float* po = a.part_o + ((size_t)u * a.n_att + c) * 8 * D;
    if (tid < GRP) {
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kLW; ++w) M = fmaxf(M, sm.u.at.mw[w][tid]);
        float l = 0.0f;
#pragma unroll
        for (int w = 0; w < kLW; ++w)
            if (sm.u.at.mw[w][tid] != -INFINITY) l += exp2f(sm.u.at.mw[w][tid] - M) * sm.u.at.lw[w][tid];
        pml[2 * tid] = M;
        pml[2 * tid + 1] = l;
    }
    for (int idx = tid; idx < GRP * D; idx += kLT) {
        const int h = idx / D, dim = idx % D;
        float s = 0.0f;
#pragma unroll
        for (int w = 0; w < kLW; ++w) s += sm.u.at.red[w][h][dim];
        po[idx] = s;
    }
    // ---- the last ATTEND of the unit merges the partials ----
    __threadfence();
    __syncthreads();
    if (tid == 0) sm.last = (atomicAdd(&a.attend_done[u], 1u) == (uint32_t)(a.n_att - 1));
    __syncthreads();
    if (!sm.last) return;
    __threadfence();
    const float* ml0 = a.part_ml + (size_t)u * a.n_att * 16;
    const float* o0 = a.part_o + (size_t)u * a.n_att * 8 * D;
    for (int idx = tid; idx < GRP * D; idx += kLT) {
        const int h = idx / D;
        float M = -INFINITY;
        for (int i = 0; i < a.n_att; ++i) {
            const float li = __ldcg(ml0 + i * 16 + 2 * h + 1);
            if (li > 0.0f) M = fmaxf(M, __ldcg(ml0 + i * 16 + 2 * h));
        }
        float num = 0.0f, den = 0.0f;
        for (int i = 0; i < a.n_att; ++i) {
            const float li = __ldcg(ml0 + i * 16 + 2 * h + 1);
            if (!(li > 0.0f)) continue;
            const float w = exp2f(__ldcg(ml0 + i * 16 + 2 * h) - M);
            den = fmaf(w, li, den);
            num = fmaf(w, __ldcg(o0 + (size_t)i * 8 * D + idx), num);
        }
        a.out[((size_t)b * Hq + g * GRP) * D + idx] = num / den;
    }
    if (tid == 0) a.sel.parity[u] = cur;  // every ATTEND of u has read the metadata
}

template <int D, int GRP>
__global__ void __launch_bounds__(kLT, 2) layer_kernel(const LayerArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    LayerSmem<D>& sm = *reinterpret_cast<LayerSmem<D>*>(smem_raw);
    const int tid = threadIdx.x;
    for (;;) {
        if (tid == 0) sm.item = (int)atomicAdd(a.ticket, 1u);
        __syncthreads();
        const int idx = sm.item;
        __syncthreads();
        if (idx >= a.n_items) break;
        const int2 it = a.items[idx];
        const int u = it.y & 0xffff, k = it.y >> 16;
#ifdef SKV_TRACE
        if (tid == 0 && idx < 2048) g_item_t[idx][0] = gtime();
#endif
        if (it.x == kItemScore)
            score_item<D, GRP>(a, sm, u, k);
        else if (it.x == kItemSelect)
            select_item<D, GRP>(a, sm, u, k);
        else
            attend_item<D, GRP>(a, sm, u, k);
        __syncthreads();
#ifdef SKV_TRACE
        if (tid == 0 && idx < 2048) g_item_t[idx][1] = gtime();
#endif
    }
    // the last CTA out returns the scratch counters to zero for the next launch
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(a.exit_count, 1u) == gridDim.x - 1) {
            const int units = a.B * a.G;
            for (int i = 0; i < units; ++i) a.score_done[i] = a.select_done[i] = a.attend_done[i] = 0u;
            *a.ticket = 0u;
            __threadfence();
            *a.exit_count = 0u;
        }
    }
}

// ------------------------------------------------------------------------------------------- host

int layer_score_items(int d, int S_b) {
    const int TS = kLTileBytes / (d * 2);
    return max(1, (S_b + kLScoreTiles * TS - 1) / (kLScoreTiles * TS));
}

int layer_attend_items(int tau) { return (tau + kLAtt - 1) / kLAtt; }

int layer_item_sentences(int d) { return kLScoreTiles * kLTileBytes / (d * 2); }

// Queue order: every SCORE first (the whole GPU streams E at once), then the SELECTs, then the
// ATTENDs chunk-major (every unit's first chunk before any second chunk), so attention of the
// units selected first starts while later selections finish.  `group` orders units within each
// phase (kept for experiments; the default interleaves nothing).
std::vector<int2> layer_schedule(const std::vector<int>& S_host, int G, int d, int tau, int group) {
    (void)group;
    const int B = (int)S_host.size(), units = B * G;
    const int n_att = layer_attend_items(tau);
    std::vector<int2> items;
    for (int u = 0; u < units; ++u)
        for (int i = 0; i < layer_score_items(d, S_host[u / G]); ++i) items.push_back(make_int2(kItemScore, u | (i << 16)));
    for (int u = 0; u < units; ++u)
        items.push_back(make_int2(kItemSelect, u | (layer_score_items(d, S_host[u / G]) << 16)));
    for (int i = 0; i < n_att; ++i)
        for (int u = 0; u < units; ++u) items.push_back(make_int2(kItemAttend, u | (i << 16)));
    return items;
}

template <int D>
static size_t smem_for(int Smax, int tau) {
    // SELECT: list offsets + (id, key, len) per candidate (<= Smax); ATTEND: tok + src
    const size_t tail = std::max((size_t)Smax * 12 + 4 * 64 + 16, sizeof(int32_t) * (2 * (size_t)tau + 1));
    return std::max(sizeof(LayerSmem<D>), LayerSmem<D>::tail_offset() + tail);
}

size_t layer_smem_bytes(int d, int Smax, int tau) { return d == 128 ? smem_for<128>(Smax, tau) : smem_for<64>(Smax, tau); }

template <int D, int GRP>
static cudaError_t launch_layer_t(const LayerArgs& a, cudaStream_t st) {
    const size_t smem = smem_for<D>(a.Smax, a.tau);
    static size_t configured = 0;
    static int grid = 0;
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(layer_kernel<D, GRP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(layer_kernel<D, GRP>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared);
        int per_sm = 0, dev = 0, sms = 0;
        if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, layer_kernel<D, GRP>, kLT, smem);
        if (e == cudaSuccess) e = cudaGetDevice(&dev);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return e;
        const char* cap = getenv("SKV_LAYER_CTAS_PER_SM");  // experiments: fewer CTAs per SM
        if (cap) per_sm = std::min(per_sm, std::max(1, atoi(cap)));
        grid = std::max(1, per_sm) * sms;  // persistent: every CTA resident
        configured = smem;
    }
    layer_kernel<D, GRP><<<grid, kLT, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_layer(const LayerArgs& a, int grp, int d, cudaStream_t st) {
#define SKV_LY(DV, GV) return launch_layer_t<DV, GV>(a, st)
    if (d == 128) {
        switch (grp) {
            case 1: SKV_LY(128, 1);
            case 2: SKV_LY(128, 2);
            case 4: SKV_LY(128, 4);
            case 8: SKV_LY(128, 8);
        }
    } else {
        switch (grp) {
            case 1: SKV_LY(64, 1);
            case 2: SKV_LY(64, 2);
            case 4: SKV_LY(64, 4);
            case 8: SKV_LY(64, 8);
        }
    }
#undef SKV_LY
    return cudaErrorInvalidValue;
}

}  // namespace skv
