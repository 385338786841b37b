// decode_fused.cu -- D2 (budgeted whole-sentence selection) fused with D3 + D4 (gather + Eq. 3
// attention) in one thread-block cluster per (b, g) unit, plus the deferred D1 state update.
//
// D2: P:444 (Sec. 4.2), Alg. 1 line 17; readings A13-A15.  D3/D4: Alg. 1
// lines 18-19; readings A16-A18.  Same arithmetic and results as select_kernel +
// attend_kernel (decode_select.cu, decode_attend.cu); this file only changes how the work is laid
// out on the GPU:
//   * the selection of a unit is spread over the kCL CTAs of its cluster: CTA r owns the
//     contiguous sentence range [r*per, (r+1)*per); key-range reduction, the 2048-bin
//     length-weighted histogram, the crossing-bin search, candidate ranking and the ordered
//     compaction are exchanged through distributed shared memory (DSMEM) with cluster barriers;
//   * while the selection runs (HBM otherwise idle), every CTA issues L2 prefetches
//     (cp.async.bulk.prefetch.L2) of its share of the K/V runs this unit selected at the previous
//     decode step -- selections change little from token to token, so the attention phase then
//     mostly reads L2;
//   * the selection metadata lands directly in every CTA's shared memory (DSMEM stores), and the
//     attention phase (attend_core.cuh) starts without another launch.
#include "device_util.cuh"
#include "skv_internal.cuh"

namespace skv {
SKV_TRACE_DEFINE(fused)
}  // namespace skv

#include "attend_core.cuh"

namespace skv {

constexpr int kFBins = 2048;
constexpr int kFCand = 1024;
constexpr int kFKeys = 4096;  // sentences per CTA held in shared memory (host checks Smax <= kCL * kFKeys)
constexpr size_t kFScratch = (size_t)kFBins * 8 + (size_t)kFCand * 12 + (size_t)kFKeys * 6;

// Dynamic shared memory: [AttSmem][tok: tau+1][srcs: tau][pad to 16][selection scratch, unless it
// fits in the (then idle) K/V stages].
template <int D, int GRP>
__host__ __device__ constexpr bool scratch_in_stages() { return kFScratch <= sizeof(AttSmem<D, GRP>::K) + sizeof(AttSmem<D, GRP>::V); }
template <int D, int GRP>
size_t fused_smem_bytes(int tau) {
    const size_t meta = (sizeof(int32_t) * (2 * (size_t)tau + 1) + 15) / 16 * 16;
    return sizeof(AttSmem<D, GRP>) + meta + (scratch_in_stages<D, GRP>() ? 0 : kFScratch);
}

__device__ __forceinline__ unsigned long long fkey64(uint32_t k, int s) {
    return ((unsigned long long)k << 32) | (unsigned long long)(0xffffffffu - (uint32_t)s);
}

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

struct FusedCtl {
    uint32_t lo, hi;             // key range (this CTA's contribution, then the cluster's)
    uint32_t cb, rem, ncb;       // crossing bin, remaining budget, sentences in the bin
    uint32_t ncand;              // candidates gathered in rank 0
    uint32_t all_fit;
    unsigned long long thr;      // select key64 > thr
    unsigned long long stot;     // this CTA's histogram-slice weight total
    unsigned long long tie_w;    // this CTA's tied weight (lo == hi path)
    unsigned long long cnt_tok;  // this CTA's selected (count << 32 | tokens)
    uint32_t red_lo, red_hi;     // block reductions
    unsigned long long ws64[32];
    uint32_t ws32[32];
};

template <int D, int GRP>
__global__ void __cluster_dims__(kCL, 1, 1) __launch_bounds__(kAttThreads, GRP <= 4 ? 2 : 1)
fused_select_attend_kernel(const float* __restrict__ scores, const int32_t* __restrict__ off, int off_stride,
                           const int32_t* __restrict__ S, int G, int Smax, int tau,
                           const __nv_bfloat16* __restrict__ q, const int32_t* __restrict__ input_token,
                           const int32_t* __restrict__ bset, int nb, float* __restrict__ Sq,
                           int32_t* __restrict__ cnt, KvSrc kv, SelBufs sel, int32_t* __restrict__ out_ids,
                           int32_t* __restrict__ out_count, int32_t* __restrict__ out_tokens,
                           float* __restrict__ out, float scale_log2) {
    constexpr int NT = kAttThreads;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    AttSmem<D, GRP>& sm = *reinterpret_cast<AttSmem<D, GRP>*>(smem_raw);
    int32_t* tok = reinterpret_cast<int32_t*>(smem_raw + sizeof(AttSmem<D, GRP>));  // [tau + 1]
    int32_t* srcs = tok + (tau + 1);                                                // [tau]
    // selection scratch: overlays the K/V stages (idle until the attention phase) when it fits
    unsigned char* scr = scratch_in_stages<D, GRP>()
                             ? reinterpret_cast<unsigned char*>(&sm.K[0][0])
                             : smem_raw + sizeof(AttSmem<D, GRP>) + (sizeof(int32_t) * (2 * (size_t)tau + 1) + 15) / 16 * 16;
    unsigned long long* hist = reinterpret_cast<unsigned long long*>(scr);  // [kFBins]
    unsigned long long* ckey = hist + kFBins;                               // [kFCand] (used in rank 0)
    uint32_t* clen = reinterpret_cast<uint32_t*>(ckey + kFCand);            // [kFCand] (used in rank 0)
    uint32_t* skey = clen + kFCand;                                          // [kFKeys]
    uint16_t* slen = reinterpret_cast<uint16_t*>(skey + kFKeys);             // [kFKeys]
    __shared__ FusedCtl ctl;
    __shared__ unsigned long long slice[kFBins / kCL];

    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int g = blockIdx.y, b = blockIdx.z;
    const int unit = b * G + g;
    const int tid = threadIdx.x, lane = tid & 31;
    const int Hq = G * GRP;
    SKV_TRACE_POINT(0);

    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&sm.bar[s], 1);
            sm.done[s] = 0u;
        }
        ctl.lo = 0xffffffffu;
        ctl.hi = 0u;
        ctl.ncand = 0u;
        ctl.all_fit = 0u;
        ctl.tie_w = 0ull;
    }
    if (tid < kAttWarps * GRP) {
        (&sm.mw[0][0])[tid] = -INFINITY;
        (&sm.lw[0][0])[tid] = 0.0f;
    }
    pdl_wait();
    SKV_TRACE_POINT(1);

    const int Sb = S[b];
    const int per = (Sb + kCL - 1) / kCL;
    const int r0 = min(Sb, rank * per), r1 = min(Sb, r0 + per);
    const int nloc = r1 - r0;
    const float* sc = scores + (size_t)unit * Smax;
    const int32_t* o = off + (size_t)b * off_stride;
    // device residency only (host checks): rows are context tokens, slot_stride == 0
    const __nv_bfloat16* Kh = kv.K + (size_t)unit * kv.unit_stride * D;
    const __nv_bfloat16* Vh = kv.V + (size_t)unit * kv.unit_stride * D;
    const int prev = sel.parity[unit], cur = prev ^ 1;
    int32_t* g_tok = sel.tok_of(cur, unit);
    int32_t* g_src = sel.src_of(cur, unit);
    int32_t* g_ids = sel.ids_of(cur, unit);

    // ---- (a) L2 prefetch of the previous step's selection (this CTA's share) ----
    {
        const int pc = *sel.count_of(prev, unit);
        const int32_t* p_tok = sel.tok_of(prev, unit);
        const int32_t* p_src = sel.src_of(prev, unit);
        const int pper = (pc + kCL - 1) / kCL;
        const int p0 = min(pc, rank * pper), p1 = min(pc, p0 + pper);
        for (int j = p0 + tid; j < p1; j += NT) {
            const int n = p_tok[j + 1] - p_tok[j];
            const size_t src = (size_t)p_src[j] * D;
            prefetch_l2(Kh + src, (uint32_t)(n * D * 2));
            prefetch_l2(Vh + src, (uint32_t)(n * D * 2));
        }
    }
    // ---- (b) deferred D1 state update (Eq. 2 sentence cache; reset at a boundary input, A11) ----
    {
        const bool reset = in_set(input_token[b], bset, nb);
        const size_t base = ((size_t)b * Hq + (size_t)g * GRP) * D;
        constexpr int E = (GRP * D + kCL - 1) / kCL;
        for (int i = rank * E + tid; i < min(GRP * D, rank * E + E); i += NT)
            Sq[base + i] = reset ? 0.0f : __fadd_rn(Sq[base + i], __bfloat162float(q[base + i]));
        if (rank == 0 && tid == 0) cnt[unit] = reset ? 0 : cnt[unit] + 1;
    }
    // ---- (c) keys and lengths of this CTA's sentences -> shared memory; local key range ----
    {
        uint32_t mn = 0xffffffffu, mx = 0u;
        for (int i = tid; i < nloc; i += NT) {
            const int s = r0 + i;
            const uint32_t k = ordered_key(sc[s]);
            skey[i] = k;
            slen[i] = (uint16_t)(o[s + 1] - o[s]);
            mn = min(mn, k);
            mx = max(mx, k);
        }
        mn = __reduce_min_sync(0xffffffffu, mn);
        mx = __reduce_max_sync(0xffffffffu, mx);
        __syncthreads();  // ctl initialised
        if (lane == 0) {
            atomicMin(&ctl.lo, mn);
            atomicMax(&ctl.hi, mx);
        }
    }
    // thread-contiguous ownership of the CTA's range for the ordered passes
    const int EL = (nloc + NT - 1) / NT;
    const int i0 = min(nloc, tid * EL), i1 = min(nloc, i0 + EL);
    SKV_TRACE_POINT(25);
    cluster.sync();  // #1: local key ranges ready
    uint32_t lo = 0xffffffffu, hi = 0u;
#pragma unroll
    for (int r = 0; r < kCL; ++r) {
        const FusedCtl* rc = cluster.map_shared_rank(&ctl, r);
        lo = min(lo, rc->lo);
        hi = max(hi, rc->hi);
    }
    uint32_t rem = (uint32_t)tau;
    bool all_fit = false;
    unsigned long long thr = 0ull;
    for (int level = 0;; ++level) {
        if (lo == hi) {
            // every remaining candidate carries key lo: ascending index decides (tie rule)
            uint32_t tw = 0;
            for (int i = i0; i < i1; ++i)
                if (skey[i] == lo) tw += slen[i];
            uint32_t ttot;
            const uint32_t tbefore = block_incl_sum<uint32_t>(tw, ctl.ws32, &ttot) - tw;
            if (tid == 0) ctl.tie_w = ttot;
            cluster.sync();
            unsigned long long before_r = 0, total = 0;
#pragma unroll
            for (int r = 0; r < kCL; ++r) {
                const unsigned long long w = cluster.map_shared_rank(&ctl, r)->tie_w;
                if (r < rank) before_r += w;
                total += w;
            }
            if (level == 0 && total <= rem) {
                all_fit = true;
                break;
            }
            const unsigned long long mybefore = before_r + tbefore;
            if (mybefore <= rem && mybefore + tw > rem) {
                unsigned long long acc = mybefore;
                for (int i = i0; i < i1; ++i) {
                    if (skey[i] != lo) continue;
                    acc += slen[i];
                    if (acc > rem) {
                        const unsigned long long t = fkey64(lo, r0 + i);
#pragma unroll
                        for (int r = 0; r < kCL; ++r) cluster.map_shared_rank(&ctl, r)->thr = t;
                        break;
                    }
                }
            }
            cluster.sync();
            thr = ctl.thr;
            break;
        }
        // ---- local length-weighted histogram over [lo, hi] (count << 32 | weight per bin) ----
        const unsigned long long span = (unsigned long long)(hi - lo) + 1ull;
        const unsigned long long mul = span >= kFBins ? ((unsigned long long)kFBins << 32) / span : 0ull;
        auto bin_of = [&](uint32_t k) -> uint32_t {
            return mul ? (uint32_t)(((unsigned long long)(k - lo) * mul) >> 32) : (k - lo);
        };
        for (int i = tid; i < kFBins; i += NT) hist[i] = 0ull;
        __syncthreads();
        for (int i = tid; i < nloc; i += NT) {
            const uint32_t k = skey[i];
            if (k < lo || k > hi) continue;
            atomicAdd(&hist[bin_of(k)], (1ull << 32) | (unsigned long long)slen[i]);
        }
        if (level == 0) SKV_TRACE_POINT(26);
        cluster.sync();  // #2: all local histograms complete
        // CTA r owns bins [r*SB, (r+1)*SB): sum them over the cluster
        constexpr int SB = kFBins / kCL;
        unsigned long long wslice = 0;
        for (int t = tid; t < SB; t += NT) {
            unsigned long long v = 0;
#pragma unroll
            for (int r = 0; r < kCL; ++r) v += cluster.map_shared_rank(hist, r)[rank * SB + t];
            slice[t] = v;
            wslice += v & 0xffffffffull;
        }
        {
            unsigned long long tot;
            block_incl_sum<unsigned long long>(wslice, ctl.ws64, &tot);
            if (tid == 0) ctl.stot = tot;
        }
        cluster.sync();  // #3: slice totals ready (local histograms may now be overwritten)
        unsigned long long above_r = 0, total = 0;
#pragma unroll
        for (int r = 0; r < kCL; ++r) {
            const unsigned long long w = cluster.map_shared_rank(&ctl, r)->stot;
            if (r > rank) above_r += w;
            total += w;
        }
        if (level == 0 && total <= rem) {
            all_fit = true;
            break;
        }
        // crossing inside this CTA's slice?  thread t holds bin rank*SB + t (SB <= NT)
        {
            const int t = tid;
            const unsigned long long v = t < SB ? slice[t] : 0ull;
            const unsigned long long w = v & 0xffffffffull;
            // weight of this slice's bins above bin t = slice total - inclusive prefix up to t
            unsigned long long stot;
            const unsigned long long incl = block_incl_sum<unsigned long long>(w, ctl.ws64, &stot);
            const unsigned long long above = above_r + (stot - incl);
            if (t < SB && above <= rem && above + w > rem) {
                const uint32_t cbv = (uint32_t)(rank * SB + t), remv = (uint32_t)(rem - above),
                               nv = (uint32_t)(v >> 32);
#pragma unroll
                for (int r = 0; r < kCL; ++r) {
                    FusedCtl* rc = cluster.map_shared_rank(&ctl, r);
                    rc->cb = cbv;
                    rc->rem = remv;
                    rc->ncb = nv;
                }
            }
        }
        if (level == 0) SKV_TRACE_POINT(27);
        cluster.sync();  // #4: crossing bin known everywhere
        const uint32_t cb = ctl.cb, ncb = ctl.ncb;
        rem = ctl.rem;
        if (ncb <= (uint32_t)kFCand) {
            // gather the crossing bin's sentences in rank 0 and rank them exactly by key64
            FusedCtl* c0 = cluster.map_shared_rank(&ctl, 0);
            unsigned long long* ck0 = cluster.map_shared_rank(ckey, 0);
            uint32_t* cl0 = cluster.map_shared_rank(clen, 0);
            for (int i = tid; i < nloc; i += NT) {
                const uint32_t k = skey[i];
                if (k < lo || k > hi || bin_of(k) != cb) continue;
                const uint32_t pos = atomicAdd(&c0->ncand, 1u);
                ck0[pos] = fkey64(k, r0 + i);
                cl0[pos] = slen[i];
            }
            cluster.sync();  // #5: candidates gathered
            if (rank == 0) {
                const int nc = (int)ctl.ncand;
                for (int c = tid; c < nc; c += NT) {
                    const unsigned long long mk = ckey[c];
                    uint32_t wabove = 0;
                    for (int j = 0; j < nc; ++j)
                        if (ckey[j] > mk) wabove += clen[j];
                    if (wabove <= rem && wabove + clen[c] > rem) {
#pragma unroll
                        for (int r = 0; r < kCL; ++r) cluster.map_shared_rank(&ctl, r)->thr = mk;
                    }
                }
            }
            if (level == 0) SKV_TRACE_POINT(28);
            cluster.sync();  // #6: threshold known everywhere
            thr = ctl.thr;
            break;
        }
        // too many candidates: narrow [lo, hi] to the crossing bin's key range and repeat
        {
            uint32_t mn = 0xffffffffu, mx = 0u;
            for (int i = tid; i < nloc; i += NT) {
                const uint32_t k = skey[i];
                if (k < lo || k > hi || bin_of(k) != cb) continue;
                mn = min(mn, k);
                mx = max(mx, k);
            }
            mn = __reduce_min_sync(0xffffffffu, mn);
            mx = __reduce_max_sync(0xffffffffu, mx);
            if (tid == 0) {
                ctl.red_lo = 0xffffffffu;
                ctl.red_hi = 0u;
            }
            __syncthreads();
            if (lane == 0) {
                atomicMin(&ctl.red_lo, mn);
                atomicMax(&ctl.red_hi, mx);
            }
        }
        cluster.sync();
        uint32_t nlo = 0xffffffffu, nhi = 0u;
#pragma unroll
        for (int r = 0; r < kCL; ++r) {
            const FusedCtl* rc = cluster.map_shared_rank(&ctl, r);
            nlo = min(nlo, rc->red_lo);
            nhi = max(nhi, rc->red_hi);
        }
        lo = nlo;
        hi = nhi;
        cluster.sync();  // everyone has read red_lo / red_hi before they can be reused
    }

    // ---- ordered compaction: ascending ids + token offsets, written to global and to every
    //      CTA's shared-memory metadata ----
    unsigned long long mine = 0;
    for (int i = i0; i < i1; ++i)
        if (all_fit || fkey64(skey[i], r0 + i) > thr) mine += (1ull << 32) | slen[i];
    unsigned long long ctot;
    const unsigned long long excl_local = block_incl_sum<unsigned long long>(mine, ctl.ws64, &ctot) - mine;
    if (tid == 0) ctl.cnt_tok = ctot;
    cluster.sync();  // #7: per-CTA selected counts ready
    unsigned long long base = 0, total = 0;
#pragma unroll
    for (int r = 0; r < kCL; ++r) {
        const unsigned long long v = cluster.map_shared_rank(&ctl, r)->cnt_tok;
        if (r < rank) base += v;
        total += v;
    }
    const int count = (int)(total >> 32);
    const int ntok = (int)(total & 0xffffffffull);
    if (mine) {
        const unsigned long long e = base + excl_local;
        int pos = (int)(e >> 32);
        int toff = (int)(e & 0xffffffffull);
        for (int i = i0; i < i1; ++i) {
            if (!(all_fit || fkey64(skey[i], r0 + i) > thr)) continue;
            const int s = r0 + i;
            const int src = o[s];
            g_ids[pos] = s;
            g_tok[pos] = toff;
            g_src[pos] = src;
            if (out_ids) out_ids[(size_t)unit * tau + pos] = s;
#pragma unroll
            for (int r = 0; r < kCL; ++r) {
                cluster.map_shared_rank(tok, r)[pos] = toff;
                cluster.map_shared_rank(srcs, r)[pos] = src;
            }
            ++pos;
            toff += slen[i];
        }
    }
    if (tid == 0) {
        tok[count] = ntok;  // every CTA writes its own copy
        if (rank == 0) {
            g_tok[count] = ntok;
            *sel.count_of(cur, unit) = count;
            if (out_count) out_count[unit] = count;
            if (out_tokens) out_tokens[unit] = ntok;
        }
    }
    if (out_ids) {
        const int tail = tau - count, tper = (tail + kCL - 1) / kCL;
        for (int i = count + rank * tper + tid; i < min(tau, count + rank * tper + tper); i += NT)
            out_ids[(size_t)unit * tau + i] = -1;
    }
    SKV_TRACE_POINT(29);
    cluster.sync();  // #8: every CTA holds the full selection metadata; scratch is dead

    attend_body<D, GRP>(sm, tok, srcs, count, Kh, Vh, q, out, b, g, G, scale_log2, cluster);
    if (rank == 0 && tid == 0) sel.parity[unit] = cur;  // all CTAs read parity before the first barrier
}

template <int D, int GRP>
static cudaError_t launch_fused_t(dim3 grid, cudaStream_t st, const float* scores, const int32_t* off, int off_stride,
                                  const int32_t* S, int G, int Smax, int tau, const __nv_bfloat16* q,
                                  const int32_t* input_token, const int32_t* bset, int nb, float* Sq, int32_t* cnt,
                                  KvSrc kv, SelBufs sel, int32_t* out_ids, int32_t* out_count, int32_t* out_tokens,
                                  float* out, float scale_log2) {
    const size_t smem = fused_smem_bytes<D, GRP>(tau);
    static size_t configured = 0;
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(fused_select_attend_kernel<D, GRP>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(fused_select_attend_kernel<D, GRP>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    return launch_pdl(fused_select_attend_kernel<D, GRP>, grid, dim3(kAttThreads), smem, st, scores, off, off_stride,
                      S, G, Smax, tau, q, input_token, bset, nb, Sq, cnt, kv, sel, out_ids, out_count, out_tokens, out,
                      scale_log2);
}

bool fused_supported(int d, int grp, int Smax, int tau) {
    (void)grp;
    return (d == 64 || d == 128) && Smax <= kCL * kFKeys && tau <= 8192;
}

cudaError_t launch_fused_select_attend(const float* scores, const int32_t* off, int off_stride, const int32_t* S,
                                       int B, int G, int grp, int d, int Smax, int tau, const __nv_bfloat16* q,
                                       const int32_t* input_token, const int32_t* bset, int nb, float* Sq,
                                       int32_t* cnt, KvSrc kv, SelBufs sel, int32_t* out_ids, int32_t* out_count,
                                       int32_t* out_tokens, float* out, cudaStream_t st) {
    dim3 grid(kCL, G, B);
    const float scale_log2 = (float)(1.0 / sqrt((double)d) * 1.4426950408889634);
#define SKV_FU(DV, GV)                                                                                              \
    return launch_fused_t<DV, GV>(grid, st, scores, off, off_stride, S, G, Smax, tau, q, input_token, bset, nb, Sq, \
                                  cnt, kv, sel, out_ids, out_count, out_tokens, out, scale_log2)
    if (d == 128) {
        switch (grp) {
            case 1: SKV_FU(128, 1);
            case 2: SKV_FU(128, 2);
            case 4: SKV_FU(128, 4);
            case 8: SKV_FU(128, 8);
        }
    } else {
        switch (grp) {
            case 1: SKV_FU(64, 1);
            case 2: SKV_FU(64, 2);
            case 4: SKV_FU(64, 4);
            case 8: SKV_FU(64, 8);
        }
    }
#undef SKV_FU
    return cudaErrorInvalidValue;
}

}  // namespace skv
