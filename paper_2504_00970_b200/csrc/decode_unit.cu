// decode_unit.cu -- one decode step of one layer, D1 + D2 + D3 + D4, in ONE launch: a
// thread-block cluster of kUC CTAs per (b, g) unit (device residency).
//
// Same arithmetic and results as score_kernel + select_kernel + attend_mma_kernel; this file only
// changes where the work runs so that a layer costs one launch and two cluster barriers:
//
//   1. score (D1; Eq. 2, S = qbar^T kbar P:440-442, Alg. 1 l.14-16): CTA r streams the
//      embeddings of its contiguous sentence range [r*chunk, (r+1)*chunk) through a TMA bulk-copy
//      ring (cp.async.bulk + mbarrier, L2 evict-first) and keeps the ordered 32-bit keys in shared
//      memory.  (L2 prefetches -- of the K/V runs selected at the previous step, of the next layer's
//      E, of this step's selection -- were measured on B200 in r01 and did not pay.)
//   2. select (D2; Alg. 1 l.17, readings A13-A15): the budgeted selection is the maximal
//      prefix of the ranking by key64 = (ordered(score) << 32) | (0xffffffff - s) whose length
//      fits tau.  Fast path: each CTA lists its sentences at or above a band around the previous
//      step's crossing point; after one cluster barrier every CTA ranks the listed band entries
//      (mode 0) or, if the weight above the band already exceeds tau, the listed entries above it
//      (mode 2).  General path (a list overflowed, or the crossing point fell below the band): each
//      CTA first cuts its own range down to *local candidates*: a sentence whose
//      local weight-above (summed lengths of the CTA's sentences ranked above it) exceeds tau can
//      never be selected, so it keeps every sentence ranked at or above its local crossing point
//      (one length-weighted 1024-bin histogram over the local key range; the crossing bin is kept
//      whole, so the list is a superset of local prefix + crossing sentence).  Claim: ranking the
//      union U of the lists is exact -- for s in U, (weight of U ranked above s) + n_s <= tau iff s
//      is selected.  (If a sentence t above s is missing from U, the crossing sentence of t's CTA and
//      everything above it are in U and above s, and they already weigh more than tau.)  After one
//      cluster barrier every CTA copies the lists (DSMEM) into its own shared memory and ranks U
//      (typically ~100 candidates per CTA instead of S/kUC sentences) by the same range-refining
//      histogram as select_kernel -- redundantly in all CTAs, so no second exchange is needed.
//      Lists are in ascending sentence order, so an ordered block scan yields the ascending ids and
//      gathered token offsets.  Rank 0 stores the selection (double-buffered SelBufs slot) and does
//      the deferred Eq. 2 state update (every CTA has read Sq before the barrier).
//   3. gather + attend (D3 + D4; Alg. 1 l.18-19): CTA r takes its 1/kUC of the 16-token
//      tiles of the gathered tokens; rows are read straight from the context K/V (one contiguous
//      run per sentence) into mma.sync fragments (mma_attend.cuh); warps merge through shared
//      memory, the kUC CTA partials through DSMEM (second cluster barrier).  (Storing the partials
//      to global memory for the unit's last CTA to combine, with a split cluster barrier so that
//      CTAs exit early, was measured slower on B200: with programmatic launch the next layer's
//      clusters then fill the freed SMs unevenly and part of the grid runs as a second wave.)
//      This phase is the non-inlined attend_phase; where one CTA per SM is all the shared memory
//      allows, the kernel is instantiated with launch bounds (256, 1) and a warp keeps two tiles in
//      flight.
// Host residency: see the page-cache comment at the row-table step (fill-in without a plan for pages
// that have a slot; the plan for pages that have none, applied by the lowest planning rank).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "device_util.cuh"
#include "mma_attend.cuh"
#include "skv_internal.cuh"

namespace cg = cooperative_groups;

namespace skv {
SKV_TRACE_DEFINE(unit)
#ifdef SKV_TRACE
// per CTA (unit * kUC + rank < 1024): SM id + globaltimer (ns) at the phase boundaries
__device__ unsigned long long g_unit_t[1024][32];
extern "C" __attribute__((visibility("default"))) int sentencekv_debug_unit(unsigned long long* out) {
    return (int)cudaMemcpyFromSymbol(out, g_unit_t, sizeof(g_unit_t));
}
// per launch (ring of 64): [0] first CTA entry, [1] first return from the programmatic-launch wait,
// [2] last CTA exit (globaltimer ns)
__device__ unsigned long long g_launch_t[64][4];
extern "C" __attribute__((visibility("default"))) int sentencekv_debug_launches(unsigned long long* out, int reset) {
    if (reset) {
        static unsigned long long init[64][4];
        for (auto& r : init) r[0] = r[1] = ~0ull, r[2] = r[3] = 0ull;
        return (int)cudaMemcpyToSymbol(g_launch_t, init, sizeof(init));
    }
    return (int)cudaMemcpyFromSymbol(out, g_launch_t, sizeof(g_launch_t));
}
__device__ __forceinline__ void launch_stamp(int idx, int which) {
    if (threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (which == 2) atomicMax(&g_launch_t[idx & 63][2], t);
        else atomicMin(&g_launch_t[idx & 63][which], t);
    }
}
#define SKV_LSTAMP(w) launch_stamp(trace_idx, (w))
__device__ __forceinline__ void unit_stamp(int cta, int ph) {
    if (threadIdx.x == 0 && cta < 1024) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_unit_t[cta][ph] = t;
        if (ph == 0) {
            unsigned int sm;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            g_unit_t[cta][23] = sm;
            g_unit_t[cta][24] = 0;
        }
    }
}
#define SKV_USTAMP(ph) unit_stamp(unit * kUC + rank, (ph))
#else
#define SKV_USTAMP(ph) \
    do {               \
    } while (0)
#define SKV_LSTAMP(w) \
    do {              \
    } while (0)
#endif

namespace {

constexpr int kUT = 256;                 // threads per CTA
constexpr int kUW = kUT / 32;
constexpr int kUC = 8;                   // CTAs per cluster (= per unit)
constexpr int kUTileBytes = 16384;       // E bytes per TMA stage
constexpr int kUStages = 3;
constexpr int kULocalCap = 2048;         // sentences per CTA (supported: Smax <= kUC * kULocalCap)
constexpr int kUOwnCap = 256;            // own candidate list kept in shared memory (else global scratch)
constexpr int kPage = 16;                // host residency: tokens per working-set page
constexpr int kNeedCap = 384;            // host residency: pages of a selection tracked by the cache plan
constexpr int kMaxPageWords = 512;       // host residency: page bitmap words (contexts up to 16384 pages)
constexpr int kMaxSlots = 1024;          // host residency: working-set pages per unit
constexpr uint32_t kEmpty = 0xffffffffu; // page-table entry of a page that is not resident
constexpr int kUBins = 1024;
// The next step's band: [crossing key - (w << kBandLoShift), lowest selected key + w], w = 2^19
// ordered-key units (~4% of a score).  Measured at 8b-128k with fresh queries (r02): the crossing
// point falls below the band far more often than above it (the scores of the sentences at the
// budget's edge drift down as Q_s grows); a 4x wider lower margin cut the general-path fallbacks
// and the step time 0.887 -> 0.866 ms (8x: lists overflow, 1.05 ms).
constexpr int kBandLoShift = 2;  // (r02, with the upper-part ranking: 8x / 16x measured 0.6 % / 4 % slower)
constexpr int kUExact = kUT;             // crossing-bin candidates ranked exactly per refinement level
constexpr int kUGather = kUStages * kUTileBytes / 16;  // candidates gathered into the (idle) ring
constexpr int kUBandCap = 256;           // band-path list entries per CTA
constexpr int kBentCap = 2 * 4 * kULocalCap / 16;  // packed band entries in the (idle) keys + offsets area
constexpr int kBandQuad = 384;           // band entries ranked by the quadratic loop (more: histogram ranking)
static_assert(kUC * kUBandCap * (16 + 4 + 4) <= kUStages * kUTileBytes, "band lists fit the ring");
using mma::kInvalid;
using mma::kTile;

template <int D>
using USmemMerge = mma::MergeSmem<D, kUW>;
static_assert(sizeof(USmemMerge<128>) <= (size_t)kUStages * kUTileBytes, "merge area aliases the E ring");

// candidate entry: (ordered key, sentence id, first context row, length)
struct Ctl {
    int own_count;      // general path: local candidates of this CTA
    int own_global;     // general path: list stored in global scratch (overflow)
    int bn;             // band path: entries of this CTA at or above the band's lower edge
    uint32_t whi, wband;  // band path: weight above the band / inside it (this CTA)
    uint32_t wnar;        // band path: weight of the band's upper part [klo_n, khi] (this CTA)
    int base[kUC + 1];  // exclusive prefix of the cluster's list sizes
    int ok, nsel, nband, count, ntok, reset, cnt0, kc_set;
    int miss_rank;      // host residency (rank 0's copy): lowest rank of the cluster that met a miss
    int mode;           // band-list ranking mode (see step 2), -1 = general path
    int below;          // general path because the crossing point fell below the band (no list overflowed)
    uint32_t WHI, WB, WN, ks, kc;
    uint32_t lo, hi, cb, rem, ncand;
    unsigned long long thr;
};

__device__ __forceinline__ unsigned long long ukey64(uint32_t k, int s) {
    return ((unsigned long long)k << 32) | (unsigned long long)(0xffffffffu - (uint32_t)s);
}

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
        : "memory");
}

// bin(k) = (k - lo) * kUBins / span as a 32.32 fixed-point multiply: monotone in k, < kUBins;
// spans below kUBins map one key per bin.
struct Binner {
    uint32_t lo;
    unsigned long long mul;
    __device__ Binner(uint32_t lo_, uint32_t hi_) : lo(lo_) {
        const unsigned long long span = (unsigned long long)(hi_ - lo_) + 1ull;
        mul = span >= kUBins ? ((unsigned long long)kUBins << 32) / span : 0ull;
    }
    __device__ __forceinline__ uint32_t operator()(uint32_t k) const {
        return mul ? (uint32_t)(((unsigned long long)(k - lo) * mul) >> 32) : (k - lo);
    }
};

// Length-weighted histogram of `hist` (kUBins, zeroed by the caller and complete on entry): the
// crossing bin, i.e. the bin b with (weight above b) <= rem < (weight above b) + w_b, and the
// budget left inside it.  Returns false if the total weight fits (no crossing bin).  Block-wide.
__device__ __forceinline__ bool crossing_bin(const uint32_t* hist, uint32_t rem, uint32_t* ws32, Ctl& ctl,
                                             uint32_t* cb_out, uint32_t* rem_out) {
    constexpr int PB = kUBins / kUT;  // bins per thread, thread t owns [PB*t, PB*t+PB)
    const int tid = threadIdx.x;
    uint32_t w[PB], sum = 0;
#pragma unroll
    for (int i = 0; i < PB; ++i) {
        w[i] = hist[PB * tid + i];
        sum += w[i];
    }
    uint32_t total;
    const uint32_t incl = block_incl_sum<uint32_t>(sum, ws32, &total);
    if (total <= rem) return false;
    uint32_t above = total - incl;  // weight of the bins above this thread's
#pragma unroll
    for (int i = PB - 1; i >= 0; --i) {
        if (above <= rem && above + w[i] > rem) {
            ctl.cb = PB * tid + i;
            ctl.rem = rem - above;
        }
        above += w[i];
    }
    __syncthreads();
    *cb_out = ctl.cb;
    *rem_out = ctl.rem;
    return true;
}

// D3 + D4 of one CTA (step 3 of unit_step_kernel): its 16-token tiles of the gathered rows ->
// mma.sync fragments -> per-warp online softmax -> CTA partial in `msm`.  Not inlined: the caller's
// state lives across this phase, and inlined it pushed the tile registers into local memory (spills
// in the tile loop, measured slower); across a call it is saved once.
//   Kd / Vd: device residency: the unit's context rows; host residency: the unit's working-set rows
//            (r >= 0), host row -(r+1) in Khu / Vhu; rows >= genL: generated rows in Kgu / Vgu (NEXT-2)
//   MISS:    some rows of this CTA come from host (they are written through into the working set)
//   GEN:     generated rows may exist (NEXT-2: when Kgu / Vgu are set)
//   PIPE:    a warp's next tile is loaded while it computes the current one (two tiles of fragment
//            registers: only when one CTA per SM leaves the kernel the registers, e.g. tau = 4096)
template <int D, int GRP, bool HOST, bool MISS, bool GEN, bool PIPE>
__device__ __noinline__ void attend_phase(const int2* __restrict__ rowtab, int tb, int te, int T0, int T1,
                                          const __nv_bfloat16* __restrict__ qg, const __nv_bfloat16* Kd,
                                          const __nv_bfloat16* Vd, const __nv_bfloat16* Khu, const __nv_bfloat16* Vhu,
                                          const __nv_bfloat16* Kgu, const __nv_bfloat16* Vgu, int genL,
                                          unsigned long long* ledger, float scale_log2,
                                          USmemMerge<D>& msm) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int gq = lane >> 2, cq = lane & 3;
    // HBM rows: r < genL context (device residency) or working-set (host residency) rows, r >= genL
    // generated rows (NEXT-2) when Kgu is set; host residency: r < 0 host row -(r+1)
    auto devK = [&](int r) -> const __nv_bfloat16* {
        return (GEN && Kgu && r >= genL) ? Kgu + (size_t)(r - genL) * D : Kd + (size_t)r * D;
    };
    auto devV = [&](int r) -> const __nv_bfloat16* {
        return (GEN && Vgu && r >= genL) ? Vgu + (size_t)(r - genL) * D : Vd + (size_t)r * D;
    };
    auto rowK = [&](int r) -> const __nv_bfloat16* {
        return (HOST && r < 0) ? Khu + (size_t)(-(r + 1)) * D : devK(r);
    };
    auto rowV = [&](int r) -> const __nv_bfloat16* {
        return (HOST && r < 0) ? Vhu + (size_t)(-(r + 1)) * D : devV(r);
    };
    unsigned long long host_bytes = 0;
    uint4 qseg[D / 32];
    mma::load_q<D, GRP>(qseg, qg, lane);
    mma::WarpAcc<D> wacc;
    wacc.init();
    // issue: the loads of a tile's rows (K: tokens gq, gq+8; V: tokens 2cq, 2cq+1, 2cq+8, 2cq+9)
    auto issue = [&](int tile, mma::TileRegs<D>& tr) {
        const int t0 = tile * kTile;
        const int2 rk0 = rowtab[t0 + gq - T0], rk1 = rowtab[t0 + gq + 8 - T0];
        const __nv_bfloat16* pv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int2 rv = rowtab[t0 + 2 * cq + (k & 1) + 8 * (k >> 1) - T0];
            pv[k] = rv.x != kInvalid ? (MISS ? rowV(rv.x) : devV(rv.x)) : nullptr;
        }
        if constexpr (MISS)
            mma::load_tile<D>(tr, rk0.x != kInvalid ? rowK(rk0.x) : nullptr,
                              rk1.x != kInvalid ? rowK(rk1.x) : nullptr, pv, lane);
        else
            mma::load_tile<D>(tr, rk0.x != kInvalid ? devK(rk0.x) : nullptr,
                              rk1.x != kInvalid ? devK(rk1.x) : nullptr, pv, lane);
    };
    // finish: QK, online softmax, PV of a loaded tile (+ host residency write-through)
    auto finish = [&](int tile, const mma::TileRegs<D>& tr) {
        const int t0 = tile * kTile;
        mma::compute_tile<D, GRP>(wacc, tr, qseg, t0 + gq < T1, t0 + gq + 8 < T1, scale_log2, lane);
        if constexpr (MISS) {
            // write-through of the rows read from host into their working-set slot
            const int2 rk0 = rowtab[t0 + gq - T0], rk1 = rowtab[t0 + gq + 8 - T0];
            int2 rv[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) rv[k] = rowtab[t0 + 2 * cq + (k & 1) + 8 * (k >> 1) - T0];
            constexpr int NU = D / 32, NVP = D / 64;
            __nv_bfloat16* Kw = const_cast<__nv_bfloat16*>(Kd);  // (host residency: the working set)
            __nv_bfloat16* Vw = const_cast<__nv_bfloat16*>(Vd);
#pragma unroll
            for (int u = 0; u < NU; ++u) {
                if (rk0.y >= 0) *reinterpret_cast<uint4*>(Kw + (size_t)rk0.y * D + mma::kseg(cq, u)) = tr.kA[u];
                if (rk1.y >= 0) *reinterpret_cast<uint4*>(Kw + (size_t)rk1.y * D + mma::kseg(cq, u)) = tr.kB[u];
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int pp = 0; pp < NVP; ++pp)
                    if (rv[k].y >= 0) *reinterpret_cast<uint4*>(Vw + (size_t)rv[k].y * D + 8 * gq + 64 * pp) = tr.vv[k][pp];
            // host bytes: K rows (counted by the cq == 0 lanes) + V rows (gq == 0 lanes)
            if (cq == 0) host_bytes += (rk0.x != kInvalid && rk0.x < 0 ? D * 2 : 0) + (rk1.x != kInvalid && rk1.x < 0 ? D * 2 : 0);
            if (gq == 0)
#pragma unroll
                for (int k = 0; k < 4; ++k) host_bytes += (rv[k].x != kInvalid && rv[k].x < 0) ? D * 2 : 0;
        }
    };
    if constexpr (PIPE) {
        mma::TileRegs<D> ta, tc;  // two tiles in flight per warp
        int tile = tb + warp;
        if (tile < te) issue(tile, ta);
        while (tile < te) {
            int nx = tile + kUW;
            if (nx < te) issue(nx, tc);
            finish(tile, ta);
            tile = nx;
            if (tile >= te) break;
            nx = tile + kUW;
            if (nx < te) issue(nx, ta);
            finish(tile, tc);
            tile = nx;
        }
    } else {  // (the same work, written out: as lambdas the host miss variant spilled more)
        for (int tile = tb + warp; tile < te; tile += kUW) {
            const int t0 = tile * kTile;
            const int2 rk0 = rowtab[t0 + gq - T0], rk1 = rowtab[t0 + gq + 8 - T0];
            int2 rv[4];
            const __nv_bfloat16* pv[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                rv[k] = rowtab[t0 + 2 * cq + (k & 1) + 8 * (k >> 1) - T0];
                pv[k] = rv[k].x != kInvalid ? (MISS ? rowV(rv[k].x) : devV(rv[k].x)) : nullptr;
            }
            mma::TileRegs<D> tr;
            if constexpr (MISS)
                mma::load_tile<D>(tr, rk0.x != kInvalid ? rowK(rk0.x) : nullptr,
                                  rk1.x != kInvalid ? rowK(rk1.x) : nullptr, pv, lane);
            else
                mma::load_tile<D>(tr, rk0.x != kInvalid ? devK(rk0.x) : nullptr,
                                  rk1.x != kInvalid ? devK(rk1.x) : nullptr, pv, lane);
            mma::compute_tile<D, GRP>(wacc, tr, qseg, t0 + gq < T1, t0 + gq + 8 < T1, scale_log2, lane);
            if constexpr (MISS) {
                // write-through of the rows read from host into their working-set slot
                constexpr int NU = D / 32, NVP = D / 64;
                __nv_bfloat16* Kw = const_cast<__nv_bfloat16*>(Kd);  // (host residency: the working set)
                __nv_bfloat16* Vw = const_cast<__nv_bfloat16*>(Vd);
#pragma unroll
                for (int u = 0; u < NU; ++u) {
                    if (rk0.y >= 0) *reinterpret_cast<uint4*>(Kw + (size_t)rk0.y * D + mma::kseg(cq, u)) = tr.kA[u];
                    if (rk1.y >= 0) *reinterpret_cast<uint4*>(Kw + (size_t)rk1.y * D + mma::kseg(cq, u)) = tr.kB[u];
                }
#pragma unroll
                for (int k = 0; k < 4; ++k)
#pragma unroll
                    for (int pp = 0; pp < NVP; ++pp)
                        if (rv[k].y >= 0) *reinterpret_cast<uint4*>(Vw + (size_t)rv[k].y * D + 8 * gq + 64 * pp) = tr.vv[k][pp];
                // host bytes: K rows (counted by the cq == 0 lanes) + V rows (gq == 0 lanes)
                if (cq == 0) host_bytes += (rk0.x != kInvalid && rk0.x < 0 ? D * 2 : 0) + (rk1.x != kInvalid && rk1.x < 0 ? D * 2 : 0);
                if (gq == 0)
#pragma unroll
                    for (int k = 0; k < 4; ++k) host_bytes += (rv[k].x != kInvalid && rv[k].x < 0) ? D * 2 : 0;
            }
        }
    }
    if constexpr (HOST) {
        // transfer ledger: host rows read by this CTA
#pragma unroll
        for (int o2 = 16; o2 >= 1; o2 >>= 1) host_bytes += __shfl_xor_sync(0xffffffffu, host_bytes, o2);
        if (lane == 0 && host_bytes) atomicAdd(ledger, host_bytes);
    }
    mma::merge_warps<D, GRP, kUW>(msm, wacc, kUT);  // the ring / gathered area is idle now
}

}  // namespace

// HGEN (host residency only): NEXT-2 generated rows exist (device residency checks gen.Kg at run time)
template <int D, int GRP, bool HOST, bool HGEN, int MINB>
__global__ void __cluster_dims__(kUC, 1, 1) __launch_bounds__(kUT, MINB)
unit_step_kernel(const __nv_bfloat16* __restrict__ q, const int32_t* __restrict__ input_token,
                 const int32_t* __restrict__ bset, int nb, float* __restrict__ Sq, int32_t* __restrict__ cnt,
                 const __nv_bfloat16* __restrict__ E, const int32_t* __restrict__ S, const int32_t* __restrict__ off,
                 int off_stride, int G, int Smax, float* __restrict__ scores, SelBufs sel, KvSrc kv, HostCache hc,
                 int4* __restrict__ cand_g, uint2* __restrict__ hint, int band_w, float* __restrict__ out,
                 int32_t* __restrict__ out_ids, int32_t* __restrict__ out_count,
                 int32_t* __restrict__ out_tokens, const int32_t* __restrict__ sid, int sid_stride, int qmode,
                 GenSrc gen, OutPeers peers, float scale_log2, int trace_idx) {
    constexpr int TPS = 4;                      // threads per sentence (scoring)
    constexpr int NPT = D / 8 / TPS;            // canonical 8-dim partials per thread (4 or 2)
    constexpr int GPW = 32 / TPS;               // sentences per warp step
    constexpr int TS = kUTileBytes / (D * 2);   // sentences per E tile
    static_assert(TS % (kUW * GPW) == 0, "tile must split evenly over the warps");
    static_assert(GRP <= 8, "heads fill the N = 8 side of the MMA");

    SKV_LSTAMP(0);
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // [ring | keys | offs | own list | band list | sel_tok | sel_src | sel_id | rowtab]; the ring is
    // reused for the gathered lists, then for the warp-merge area
    __nv_bfloat16* ring = reinterpret_cast<__nv_bfloat16*>(smem_raw);
    int4* gath = reinterpret_cast<int4*>(smem_raw);
    USmemMerge<D>& msm = *reinterpret_cast<USmemMerge<D>*>(smem_raw);
    uint32_t* keys = reinterpret_cast<uint32_t*>(smem_raw + kUStages * kUTileBytes);
    int32_t* offs = reinterpret_cast<int32_t*>(keys + kULocalCap);
    int4* own = reinterpret_cast<int4*>(offs + kULocalCap + 4);
    int4* blist = own + kUOwnCap;
    const int tau = sel.tau;
    int32_t* sel_tok = reinterpret_cast<int32_t*>(blist + kUBandCap);  // [tau + 1]
    int32_t* sel_src = sel_tok + (tau + 1);                              // [tau]
    int32_t* sel_id = sel_src + tau;                                     // [tau]
    int2* rowtab = reinterpret_cast<int2*>(sel_tok + (3 * tau + 5) / 4 * 4);  // [rows per CTA] (source, write-through row)
    // host residency: the page-cache plan of this step, in the keys / offsets area (local to this CTA
    // and idle once the selection is made; the ring holds the merge area that other CTAs read)
    int* need = reinterpret_cast<int*>(keys);                            // [kNeedCap] pages of the selection
    uint32_t* pslot = reinterpret_cast<uint32_t*>(need + kNeedCap);     // [kNeedCap] their page-table entries
    int* slotof = reinterpret_cast<int*>(pslot + kNeedCap);             // [kNeedCap] slot this step (-1 none)
    uint32_t* rowbits = reinterpret_cast<uint32_t*>(slotof + kNeedCap); // [kNeedCap] selected rows
    int* newj = reinterpret_cast<int*>(rowbits + kNeedCap);             // [kNeedCap] non-resident pages
    int* frees = newj + kNeedCap;                                       // [kNeedCap] their slots
    uint32_t* pbits = reinterpret_cast<uint32_t*>(frees + kNeedCap);    // [kMaxPageWords] pages of the selection
    uint32_t* pbase = pbits + kMaxPageWords;                            // [kMaxPageWords] rank of each word's first page
    static_assert(kNeedCap * 24 + kMaxPageWords * 8 <= kULocalCap * 8, "plan fits the keys + offsets area");

    __shared__ uint64_t bar[kUStages];
    __shared__ float qt[D];
    __shared__ float sqsum[GRP * D];  // Sq + q_t of this step (the Eq. 2 state update, stored by rank 0)
    __shared__ uint32_t hist[kUBins];
    __shared__ uint32_t ws32[32];
    __shared__ unsigned long long ws64[32];
    __shared__ unsigned long long ckey[kUExact];
    __shared__ uint32_t clen[kUExact];
    __shared__ Ctl ctl;
    __shared__ const int4* lists[kUC];
    __shared__ int n_need_s, last_slot_s;
    __shared__ uint32_t inuse[HOST ? kMaxSlots / 32 : 1];  // host residency: slots read by this step

    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int g = blockIdx.y, b = blockIdx.z;
    const int unit = b * G + g;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int Hq = G * GRP;

    if (tid == 0) {
        for (int i = 0; i < kUStages; ++i) mbar_init(&bar[i], 1);
        ctl.lo = 0xffffffffu;
        ctl.hi = 0u;
        ctl.bn = 0;
        ctl.whi = 0u;
        ctl.wband = 0u;
        ctl.wnar = 0u;
        ctl.ks = 0xffffffffu;
        ctl.kc_set = 0;
        ctl.nsel = 0;
        ctl.nband = 0;
        ctl.ntok = 0;
        ctl.miss_rank = kUC;
    }
    // The prompt's sentence counts and embeddings are written only by the prefill, never by the
    // decode kernel this one may overlap (programmatic launch), so the first E tiles are requested
    // before waiting for it; everything the previous step wrote is read after pdl_wait().
    const int Sb = S[b];
    const int chunk = (Sb + kUC - 1) / kUC;
    const int s0 = min(Sb, rank * chunk), s1 = min(Sb, s0 + chunk);
    const int n = s1 - s0;
    const int ntiles = (n + TS - 1) / TS;
    const __nv_bfloat16* Eu = E + ((size_t)unit * Smax) * D;
    const int32_t* o = off + (size_t)b * off_stride;

    // ---------------------------------------------------------------- 1. score (D1)
    if (tid == 0) {
        const uint64_t pol = policy_evict_first();
        for (int i = 0; i < kUStages && i < ntiles; ++i) {
            const int ts = s0 + i * TS, m = min(TS, s1 - ts);
            mbar_arrive_expect_tx(&bar[i], (uint32_t)(m * D * 2));
            bulk_g2s_hint(ring + (size_t)i * TS * D, Eu + (size_t)ts * D, (uint32_t)(m * D * 2), &bar[i], pol);
        }
    }
    pdl_wait();
    SKV_TRACE_POINT(0);
    SKV_USTAMP(0);
    SKV_LSTAMP(1);
    const int prev = sel.parity[unit], cur = prev ^ 1;
    const uint2 band = hint[unit];  // [klo, khi]: where the crossing point was at the previous step
    const uint32_t klo = band.x, khi = band.y;
    // the band's upper part [klo_n, khi], klo_n = crossing point - w: the crossing point usually stays
    // there, and then only that part is ranked (the quadratic rank is ~9x cheaper than over the band)
    auto klo_narrow = [&]() -> uint32_t {
        return klo ? klo + (((uint32_t)band_w << kBandLoShift) - (uint32_t)band_w) : 0u;
    };
    if (warp == kUW - 2) {
        // does this step's input token end a sentence (Q_s reset after this step, A11)?
        const int it = input_token[b];
        const bool hit = (lane < nb && bset[lane] == it) || (lane + 32 < nb && bset[lane + 32] == it);
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (lane == 0) ctl.reset = m ? 1 : 0;
    }
    // first context row of every local sentence (+ the end of the last)
    for (int i = tid; i <= n; i += kUT) offs[i] = o[s0 + i];
    // group query of this step: qbar_h = (Sq_h + q_h) / (cnt + 1) (the appended, not yet stored,
    // Q_s), qt_g = ascending-h fp32 sum (canonical order, A23)
    if (tid < D) {
        const int c0 = cnt[unit];
        const float c = (float)(c0 + 1);
        float sv[GRP], qv[GRP];
#pragma unroll
        for (int h = 0; h < GRP; ++h) {
            const size_t idx = ((size_t)b * Hq + g * GRP + h) * D + tid;
            sv[h] = Sq[idx];
            qv[h] = __bfloat162float(q[idx]);
        }
        float acc = 0.0f;
#pragma unroll
        for (int h = 0; h < GRP; ++h) {
            const float sum = __fadd_rn(sv[h], qv[h]);
            sqsum[h * D + tid] = sum;
            const float qb = qmode ? qv[h] : __fdiv_rn(sum, c);  // qmode 1: current token's query (NEXT-3)
            acc = h == 0 ? qb : __fadd_rn(acc, qb);
        }
        qt[tid] = acc;
        if (tid == 0) ctl.cnt0 = c0;
    }
    __syncthreads();
    {
        // Canonical dot (A23): d/8 partials p_l = q[8l..8l+7] . e[8l..8l+7] (mul, then 7 fma), then
        // the tree of the xor butterfly with offsets d/16, ..., 1.  Here a sentence has TPS = 4
        // threads; thread j holds the partials l = j, j+4, (j+8, j+12): the first tree levels are
        // local adds in the same pairing, the last two are shuffles (offsets 2 and 1) -- the same
        // additions in the same order, so the score is bit-identical to the 16-lane form.
        const int j = lane % TPS, gw = lane / TPS;
        float qr[NPT][8];
#pragma unroll
        for (int c = 0; c < NPT; ++c)
#pragma unroll
            for (int i = 0; i < 8; ++i) qr[c][i] = qt[8 * (j + TPS * c) + i];
        float* sc_out = scores + (size_t)unit * Smax;
        uint32_t mn = 0xffffffffu, mx = 0u;
        for (int it = 0; it < ntiles; ++it) {
            const int st = it % kUStages;
            mbar_wait(&bar[st], (it / kUStages) & 1);
            const __nv_bfloat16* tile = ring + (size_t)st * TS * D;
            const int ts = it * TS, m = min(TS, n - ts);  // local index of the tile's first sentence
#pragma unroll
            for (int jj = 0; jj < TS / (kUW * GPW); ++jj) {
                const int r = (jj * kUW + warp) * GPW + gw;
                float pp[NPT];
#pragma unroll
                for (int c = 0; c < NPT; ++c) {
                    float f[8];
                    unpack8(*reinterpret_cast<const uint4*>(tile + (size_t)r * D + 8 * (j + TPS * c)), f);
                    float p = __fmul_rn(qr[c][0], f[0]);
#pragma unroll
                    for (int i = 1; i < 8; ++i) p = __fmaf_rn(qr[c][i], f[i], p);
                    pp[c] = p;
                }
                float p;
                if constexpr (NPT == 4) {  // d = 128: levels 8 and 4 are local
                    p = __fadd_rn(__fadd_rn(pp[0], pp[2]), __fadd_rn(pp[1], pp[3]));
                } else {                   // d = 64: level 4 is local
                    p = __fadd_rn(pp[0], pp[1]);
                }
                p = __fadd_rn(p, __shfl_xor_sync(0xffffffffu, p, 2));
                p = __fadd_rn(p, __shfl_xor_sync(0xffffffffu, p, 1));
                if (j == 0 && r < m) {
                    const int i = ts + r;
                    const uint32_t k = ordered_key(p);
                    keys[i] = k;
                    sc_out[s0 + i] = p;
                    mn = min(mn, k);
                    mx = max(mx, k);
                }
            }
            __syncthreads();  // stage st fully read
            if (tid == 0 && it + kUStages < ntiles) {
                const int tn = s0 + (it + kUStages) * TS, nn = min(TS, s1 - tn);
                mbar_arrive_expect_tx(&bar[st], (uint32_t)(nn * D * 2));
                bulk_g2s_hint(ring + (size_t)st * TS * D, Eu + (size_t)tn * D, (uint32_t)(nn * D * 2), &bar[st],
                              policy_evict_first());
            }
        }
        mn = __reduce_min_sync(0xffffffffu, mn);
        mx = __reduce_max_sync(0xffffffffu, mx);
        if (lane == 0 && n > 0) {
            atomicMin(&ctl.lo, mn);
            atomicMax(&ctl.hi, mx);
        }
    }
    __syncthreads();
    // band list (ascending sentence order): everything at or above the band's lower edge, with the
    // weights above the band and inside it
    const int per_t = (n + kUT - 1) / kUT;
    const int i0 = min(n, tid * per_t), i1 = min(n, i0 + per_t);
    {
        uint32_t mine = 0, whi = 0, wband = 0, wnar = 0;
        const uint32_t klo_n = klo_narrow();
        for (int i = i0; i < i1; ++i) {
            const uint32_t k = keys[i];
            if (k >= klo) {
                ++mine;
                const uint32_t len = (uint32_t)(offs[i + 1] - offs[i]);
                if (k > khi) whi += len;
                else {
                    wband += len;
                    if (k >= klo_n) wnar += len;
                }
            }
        }
        uint32_t total;
        uint32_t pos = block_incl_sum<uint32_t>(mine, ws32, &total) - mine;
        for (int i = i0; i < i1 && pos < (uint32_t)kUBandCap; ++i)
            if (keys[i] >= klo) blist[pos++] = make_int4((int)keys[i], s0 + i, offs[i], offs[i + 1] - offs[i]);
        whi = __reduce_add_sync(0xffffffffu, whi);
        wband = __reduce_add_sync(0xffffffffu, wband);
        wnar = __reduce_add_sync(0xffffffffu, wnar);
        if (lane == 0) {
            atomicAdd(&ctl.whi, whi);
            atomicAdd(&ctl.wband, wband);
            atomicAdd(&ctl.wnar, wnar);
        }
        if (tid == 0) ctl.bn = (int)total;
    }
    __syncthreads();
    SKV_USTAMP(1);
    cluster.sync();  // #A: band lists and counters of every CTA are complete; every CTA has read Sq
    SKV_USTAMP(2);

    // ---------------------------------------------------------------- 2. select (D2)
    // Fast path: the crossing point lies in the band [klo, khi] around the previous step's (the
    // ranking changes little from token to token): everything above khi is selected and only the
    // band is ranked.  Exact whenever its conditions hold; otherwise the general path below.
    if (warp == 0) {
        uint32_t whi = 0, wband = 0, wnar = 0;
        int bn = 0;
        const int4* lp = nullptr;
        if (lane < kUC) {
            Ctl* rc = cluster.map_shared_rank(&ctl, lane);
            whi = rc->whi;
            wband = rc->wband;
            wnar = rc->wnar;
            bn = rc->bn;
            lp = cluster.map_shared_rank(blist, lane);
        }
        const bool ovf = __any_sync(0xffffffffu, bn > kUBandCap);
        const int incl = warp_incl_sum<int>(bn);
        const uint32_t WHI = __reduce_add_sync(0xffffffffu, whi), WB = __reduce_add_sync(0xffffffffu, wband);
        const uint32_t WN = __reduce_add_sync(0xffffffffu, wnar);
        if (lane < kUC) {
            ctl.base[lane + 1] = incl;
            lists[lane] = lp;
        }
        if (lane == 0) {
            ctl.base[0] = 0;
            ctl.WHI = WHI;
            ctl.WB = WB;
            ctl.WN = WN;
            // 0: the crossing point is in the band; 2: above it (only entries above khi can be
            // selected, and all of them are listed); -1: a list overflowed, or the crossing point is
            // below the band -> general path.  (Rebuilding the lists below the band instead was
            // measured slower than the general path: its candidate set is as large and the band
            // ranking is quadratic in it.)
            int mode = -1;
            if (!ovf) {
                if (WHI <= (uint32_t)tau && (WHI + WB > (uint32_t)tau || klo == 0u)) mode = 0;
                else if (WHI > (uint32_t)tau) mode = 2;
            }
            ctl.mode = mode;
            ctl.ok = mode >= 0;
            ctl.below = (!ovf && mode < 0) ? 1 : 0;  // (then WHI + WB <= tau and klo > 0)
#ifdef SKV_TRACE
            if (unit * kUC + rank < 1024) {
                g_unit_t[unit * kUC + rank][10] = (ovf ? 1 : 0) | (WHI > (uint32_t)tau ? 2 : 0) |
                                                  (WHI + WB <= (uint32_t)tau && klo != 0u ? 4 : 0) | ((mode + 1) << 4);
                g_unit_t[unit * kUC + rank][13] = (unsigned long long)incl;
            }
#endif
        }
    }
    __syncthreads();
    SKV_USTAMP(16);
    int mode = ctl.mode;
    // ranking of the gathered lists: entries with key > auto_gt are selected, entries with key in
    // [rank_ge, auto_gt] are ranked on top of the weight W0 of everything above them, the rest is
    // not selected
    uint32_t auto_gt = khi, rank_ge = klo, W0 = ctl.WHI;
    if (mode == 2) {  // WHI > tau: the crossing point is above the band, among the listed entries > khi
        auto_gt = 0xffffffffu;
        rank_ge = khi + 1u;  // khi < 0xffffffff here (else WHI = 0)
        W0 = 0u;
    } else if (mode == 0 && klo_narrow() > klo) {
        const uint32_t klo_n = klo_narrow();
        if (ctl.WHI + ctl.WN > (uint32_t)tau) {
            rank_ge = klo_n;  // the crossing point is in the upper part: the lower part is not selected
        } else {
            auto_gt = klo_n - 1u;  // the upper part is selected too; the crossing point is below it
            W0 = ctl.WHI + ctl.WN;
        }
    }
    bool ok = mode >= 0;
    if (ok) {
        // gather the lists in rank order (so in ascending sentence order); band entries are ranked
        const int ntot = ctl.base[kUC];
        int* bidx = reinterpret_cast<int*>(gath + kUC * kUBandCap);  // [ntot] indices of band entries
        int* flag = bidx + kUC * kUBandCap;                          // [ntot] selected
        for (int i0 = tid; i0 < ntot; i0 += 4 * kUT) {
            int4 e[4];  // remote (DSMEM) loads issued together, then stored
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int i = i0 + k * kUT;
                if (i < ntot) {
                    int j = 0;
                    while (i >= ctl.base[j + 1]) ++j;
                    e[k] = lists[j][i - ctl.base[j]];
                }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int i = i0 + k * kUT;
                if (i < ntot) {
                    gath[i] = e[k];
                    const bool above = (uint32_t)e[k].x > auto_gt;
                    flag[i] = above ? 1 : 0;
                    if (!above && (uint32_t)e[k].x >= rank_ge) {
                        // band entry: its index, and (key, ~id, length) packed for the rank loop
                        const int x = atomicAdd(&ctl.nband, 1);
                        bidx[x] = i;
                        if (x < kBentCap)
                            reinterpret_cast<uint4*>(keys)[x] =
                                make_uint4((uint32_t)e[k].x, 0xffffffffu - (uint32_t)e[k].y, (uint32_t)e[k].w, 0u);
                    }
                }
            }
        }
        __syncthreads();
        SKV_USTAMP(17);
        // a band entry is selected iff (weight above the band) + (weight of band entries ranked above
        // it) + its length fits tau; the one that first does not fit is the crossing point.  Small
        // bands: every entry counts the weight above it (quadratic, no barrier).  Large bands (many
        // short buckets, e.g. after NEXT-1 retention: measured 24.6 us for the quadratic loop): the
        // range-refining length histogram of the general path over the band entries, O(n) per level.
        const int nbd = ctl.nband;
        bool quad = nbd <= kBandQuad;
        if (!quad) {
            const int per_b = (nbd + kUT - 1) / kUT;
            const int x0 = min(nbd, tid * per_b), x1 = min(nbd, x0 + per_b);
            if (tid == 0) {
                ctl.lo = 0xffffffffu;
                ctl.hi = 0u;
            }
            __syncthreads();
            {
                uint32_t mn = 0xffffffffu, mx = 0u;
                for (int x = x0; x < x1; ++x) {
                    const uint32_t k = (uint32_t)gath[bidx[x]].x;
                    mn = min(mn, k);
                    mx = max(mx, k);
                }
                mn = __reduce_min_sync(0xffffffffu, mn);
                mx = __reduce_max_sync(0xffffffffu, mx);
                if (lane == 0) {
                    atomicMin(&ctl.lo, mn);
                    atomicMax(&ctl.hi, mx);
                }
            }
            __syncthreads();
            uint32_t lo = ctl.lo, hi = ctl.hi, rem = (uint32_t)tau - W0;
            bool all_fit = false, done = false;
            unsigned long long thr = 0ull;
            for (int level = 0; level < 4 && !done; ++level) {
                for (int i = tid; i < kUBins; i += kUT) hist[i] = 0u;
                __syncthreads();
                const Binner bin(lo, hi);
                for (int x = x0; x < x1; ++x) {
                    const int4 e = gath[bidx[x]];
                    const uint32_t k = (uint32_t)e.x;
                    if (k >= lo && k <= hi) atomicAdd(&hist[bin(k)], (uint32_t)e.w);
                }
                __syncthreads();
                uint32_t cb, rem_in;
                if (!crossing_bin(hist, rem, ws32, ctl, &cb, &rem_in)) {  // (level 0 only) every entry fits
                    all_fit = true;
                    break;
                }
                if (tid == 0) {
                    ctl.lo = 0xffffffffu;
                    ctl.hi = 0u;
                    ctl.ncand = 0u;
                }
                __syncthreads();
                {
                    uint32_t mn = 0xffffffffu, mx = 0u;
                    for (int x = x0; x < x1; ++x) {
                        const int4 e = gath[bidx[x]];
                        const uint32_t k = (uint32_t)e.x;
                        if (k < lo || k > hi || bin(k) != cb) continue;
                        mn = min(mn, k);
                        mx = max(mx, k);
                        const uint32_t p = atomicAdd(&ctl.ncand, 1u);
                        if (p < (uint32_t)kUExact) {
                            ckey[p] = ukey64(k, e.y);
                            clen[p] = (uint32_t)e.w;
                        }
                    }
                    mn = __reduce_min_sync(0xffffffffu, mn);
                    mx = __reduce_max_sync(0xffffffffu, mx);
                    if (lane == 0) {
                        atomicMin(&ctl.lo, mn);
                        atomicMax(&ctl.hi, mx);
                    }
                }
                __syncthreads();
                const int nc = (int)ctl.ncand;
                if (nc <= kUExact) {  // rank the crossing bin's entries exactly (unique key64s)
                    if (tid < nc) {
                        const unsigned long long mk = ckey[tid];
                        uint32_t wab = 0;
                        for (int c = 0; c < nc; ++c)
                            if (ckey[c] > mk) wab += clen[c];
                        if (wab <= rem_in && wab + clen[tid] > rem_in) ctl.thr = mk;
                    }
                    __syncthreads();
                    thr = ctl.thr;
                    done = true;
                    break;
                }
                rem = rem_in;
                lo = ctl.lo;
                hi = ctl.hi;
                __syncthreads();
                if (lo == hi) break;  // > kUExact entries tie on one score: the quadratic rank below
            }
            if (all_fit || done) {
                for (int x = x0; x < x1; ++x) {
                    const int i = bidx[x];
                    const int4 e = gath[i];
                    if (all_fit || ukey64((uint32_t)e.x, e.y) > thr) flag[i] = 1;
                }
                if (tid == 0 && !all_fit) {
                    ctl.kc = (uint32_t)(thr >> 32);  // the crossing sentence
                    ctl.kc_set = 1;
                }
            } else {
                quad = true;
            }
        }
        if (quad) {
            const uint32_t WHI = W0;
            // band entries packed as (key, ~id, length) in the idle keys/offsets area, so the
            // quadratic rank loop reads one broadcast 16-byte word per entry, no indirection
            const uint4* bent = reinterpret_cast<const uint4*>(keys);  // packed by the gather above
            const bool packed = nbd <= kBentCap;
            for (int x = tid; x < nbd; x += kUT) {
                const int i = bidx[x];
                const int4 e = gath[i];
                const unsigned long long ke = ukey64((uint32_t)e.x, e.y);
                uint32_t w = WHI;
                if (packed) {
#pragma unroll 4
                    for (int c = 0; c < nbd; ++c) {
                        const uint4 f = bent[c];
                        if ((((unsigned long long)f.x << 32) | f.y) > ke) w += f.z;
                    }
                } else {
                    for (int c = 0; c < nbd; ++c) {
                        const int4 f = gath[bidx[c]];
                        if (ukey64((uint32_t)f.x, f.y) > ke) w += (uint32_t)f.w;
                    }
                }
                if (w + (uint32_t)e.w <= (uint32_t)tau) {
                    flag[i] = 1;
                } else if (w <= (uint32_t)tau) {
                    ctl.kc = (uint32_t)e.x;  // the crossing sentence (unique)
                    ctl.kc_set = 1;
                }
            }
        }
        __syncthreads();
        SKV_USTAMP(18);
        // ordered compaction: ascending ids and gathered token offsets
        const int pc_ = (ntot + kUT - 1) / kUT;
        const int c0 = min(ntot, tid * pc_), c1 = min(ntot, c0 + pc_);
        unsigned long long mine = 0;
        uint32_t kmin = 0xffffffffu;
        for (int i = c0; i < c1; ++i)
            if (flag[i]) {
                const int4 e = gath[i];
                mine += (1ull << 32) | (uint32_t)e.w;
                kmin = min(kmin, (uint32_t)e.x);
            }
        unsigned long long tot;
        const unsigned long long excl = block_incl_sum<unsigned long long>(mine, ws64, &tot) - mine;
        int pos = (int)(excl >> 32);
        int32_t toff = (int32_t)(excl & 0xffffffffull);
        for (int i = c0; i < c1; ++i)
            if (flag[i]) {
                const int4 e = gath[i];
                sel_tok[pos] = toff;
                sel_src[pos] = e.z;
                sel_id[pos] = e.y;
                ++pos;
                toff += e.w;
            }
        kmin = __reduce_min_sync(0xffffffffu, kmin);
        if (lane == 0 && kmin != 0xffffffffu) atomicMin(&ctl.ks, kmin);
        if (tid == 0) {
            const int count = (int)(tot >> 32);
            ctl.count = count;
            ctl.ntok = (int)(tot & 0xffffffffull);
            sel_tok[count] = ctl.ntok;
        }
        __syncthreads();
#ifdef SKV_TRACE
        if (tid == 0 && unit * kUC + rank < 1024) {
            g_unit_t[unit * kUC + rank][11] = ctl.nband;
            g_unit_t[unit * kUC + rank][12] = ctl.count;
        }
#endif
    }
    SKV_USTAMP(3);
    if (!ok) {
        // ------------------------------------------------------------ general path
        // 2a. local candidates.  When the crossing point fell below the band (no list overflowed), every
        // sentence at or above klo is selected (they weigh WHI + WB <= tau and rank above the rest):
        // the problem shrinks to the keys below klo with the budget left, rem0 = tau - (WHI + WB) --
        // the same cut and exact ranking over them; the sentences at or above klo join the lists
        // (selected by the compaction's key64 > thr like any entry ranked above the crossing)
        const bool below = ctl.below != 0;
        const uint32_t rem0 = below ? (uint32_t)tau - (ctl.WHI + ctl.WB) : (uint32_t)tau;
        for (int i = tid; i < kUBins; i += kUT) hist[i] = 0u;
        __syncthreads();
        {
            const uint32_t hi_b = below ? min(ctl.hi, klo - 1u) : ctl.hi;  // ranked keys: [ctl.lo, hi_b]
            const bool any_b = n > 0 && ctl.lo <= hi_b;
            const Binner bin(ctl.lo, any_b ? hi_b : ctl.lo);
            auto ranked = [&](uint32_t k) { return any_b && k <= hi_b; };
            for (int i = i0; i < i1; ++i)
                if (ranked(keys[i])) atomicAdd(&hist[bin(keys[i])], (uint32_t)(offs[i + 1] - offs[i]));
            __syncthreads();
            uint32_t cb = 0, rem_unused;
            const bool cross = crossing_bin(hist, rem0, ws32, ctl, &cb, &rem_unused);
            // keep bins >= cb (all sentences if the CTA's total fits) and (below) every key >= klo, in
            // ascending sentence order
            auto keep = [&](uint32_t k) { return !ranked(k) || !cross || bin(k) >= cb; };
            uint32_t mine = 0;
            for (int i = i0; i < i1; ++i) mine += keep(keys[i]) ? 1u : 0u;
            uint32_t total;
            const uint32_t excl = block_incl_sum<uint32_t>(mine, ws32, &total) - mine;
            const bool to_global = total > (uint32_t)kUOwnCap;
            int4* dst = to_global ? cand_g + ((size_t)unit * kUC + rank) * kULocalCap : own;
            uint32_t pos = excl;
            for (int i = i0; i < i1; ++i) {
                const uint32_t k = keys[i];
                if (keep(k)) dst[pos++] = make_int4((int)k, s0 + i, offs[i], offs[i + 1] - offs[i]);
            }
            if (tid == 0) {
                ctl.own_count = (int)total;
                ctl.own_global = to_global ? 1 : 0;
#ifdef SKV_TRACE
                if (unit * kUC + rank < 1024) g_unit_t[unit * kUC + rank][14] = total | (to_global ? (1ull << 32) : 0ull);
#endif
            }
        }
        cluster.sync();  // #1: every CTA's candidate list is complete
        SKV_USTAMP(4);

        // 2b. gather the lists
        if (warp == 0) {
            int c = 0;
            const int4* lp = nullptr;
            if (lane < kUC) {
                Ctl* rc = cluster.map_shared_rank(&ctl, lane);
                c = rc->own_count;
                lp = rc->own_global ? cand_g + ((size_t)unit * kUC + lane) * kULocalCap
                                    : cluster.map_shared_rank(own, lane);
            }
            const int incl = warp_incl_sum<int>(c);
            if (lane < kUC) {
                ctl.base[lane + 1] = incl;
                lists[lane] = lp;
            }
            if (lane == 0) ctl.base[0] = 0;
        }
        __syncthreads();
        const int ntot = ctl.base[kUC];
        const bool gathered = ntot <= kUGather;
#ifdef SKV_TRACE
        if (tid == 0 && unit * kUC + rank < 1024) g_unit_t[unit * kUC + rank][15] = (unsigned long long)ntot;
#endif
        if (gathered) {
            for (int i0 = tid; i0 < ntot; i0 += 4 * kUT) {
                int4 e[4];  // remote (DSMEM / global) loads issued together, then stored
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int i = i0 + k * kUT;
                    if (i < ntot) {
                        int j = 0;
                        while (i >= ctl.base[j + 1]) ++j;
                        e[k] = lists[j][i - ctl.base[j]];
                    }
                }
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (i0 + k * kUT < ntot) gath[i0 + k * kUT] = e[k];
            }
        }
        auto cand = [&](int i) -> int4 {
            if (gathered) return gath[i];
            int j = 0;
            while (i >= ctl.base[j + 1]) ++j;
            return lists[j][i - ctl.base[j]];
        };
        if (tid == 0) {
            ctl.lo = 0xffffffffu;
            ctl.hi = 0u;
        }
        __syncthreads();
        SKV_USTAMP(19);
        const int per_c = (ntot + kUT - 1) / kUT;
        const int c0 = min(ntot, tid * per_c), c1 = min(ntot, c0 + per_c);
        {
            uint32_t mn = 0xffffffffu, mx = 0u;
            for (int i = c0; i < c1; ++i) {
                const uint32_t k = (uint32_t)cand(i).x;
                if (below && k >= klo) continue;  // selected; not ranked
                mn = min(mn, k);
                mx = max(mx, k);
            }
            mn = __reduce_min_sync(0xffffffffu, mn);
            mx = __reduce_max_sync(0xffffffffu, mx);
            if (lane == 0 && c0 < c1) {
                atomicMin(&ctl.lo, mn);
                atomicMax(&ctl.hi, mx);
            }
        }
        __syncthreads();
        SKV_USTAMP(20);

        // 2c. exact selection over the union of the lists
        uint32_t lo = ctl.lo, hi = ctl.hi, rem = rem0;
        bool all_fit = lo > hi;  // (below: nothing under klo -- everything listed is selected)
        unsigned long long thr = 0;  // select key64 > thr
        for (int level = 0; !all_fit; ++level) {
            if (lo == hi) {
                // the remaining contenders all carry key lo: ascending sentence order decides (A14)
                uint32_t tw = 0;
                for (int i = c0; i < c1; ++i) {
                    const int4 e = cand(i);
                    if ((uint32_t)e.x == lo) tw += (uint32_t)e.w;
                }
                uint32_t ttot;
                const uint32_t before = block_incl_sum<uint32_t>(tw, ws32, &ttot) - tw;
                if (level == 0 && ttot <= rem) {
                    all_fit = true;
                    break;
                }
                if (before <= rem && before + tw > rem) {
                    uint32_t acc = before;
                    for (int i = c0; i < c1; ++i) {
                        const int4 e = cand(i);
                        if ((uint32_t)e.x != lo) continue;
                        acc += (uint32_t)e.w;
                        if (acc > rem) {
                            ctl.thr = ukey64(lo, e.y);
                            break;
                        }
                    }
                }
                __syncthreads();
                thr = ctl.thr;
                break;
            }
            for (int i = tid; i < kUBins; i += kUT) hist[i] = 0u;
            __syncthreads();
            const Binner bin(lo, hi);
            for (int i = c0; i < c1; ++i) {
                const int4 e = cand(i);
                const uint32_t k = (uint32_t)e.x;
                if (k >= lo && k <= hi) atomicAdd(&hist[bin(k)], (uint32_t)e.w);
            }
            __syncthreads();
            uint32_t cb, rem_in;
            if (!crossing_bin(hist, rem, ws32, ctl, &cb, &rem_in)) {
                // only possible at level 0 (the crossing bin of a level above holds more than rem)
                all_fit = true;
                break;
            }
            rem = rem_in;
            if (tid == 0) {
                ctl.lo = 0xffffffffu;
                ctl.hi = 0u;
                ctl.ncand = 0u;
            }
            __syncthreads();
            {
                uint32_t mn = 0xffffffffu, mx = 0u;
                for (int i = c0; i < c1; ++i) {
                    const int4 e = cand(i);
                    const uint32_t k = (uint32_t)e.x;
                    if (k < lo || k > hi || bin(k) != cb) continue;
                    mn = min(mn, k);
                    mx = max(mx, k);
                    const uint32_t p = atomicAdd(&ctl.ncand, 1u);
                    if (p < (uint32_t)kUExact) {
                        ckey[p] = ukey64(k, e.y);
                        clen[p] = (uint32_t)e.w;
                    }
                }
                mn = __reduce_min_sync(0xffffffffu, mn);
                mx = __reduce_max_sync(0xffffffffu, mx);
                if (lane == 0) {
                    atomicMin(&ctl.lo, mn);
                    atomicMax(&ctl.hi, mx);
                }
            }
            __syncthreads();
            if (ctl.ncand <= (uint32_t)kUExact) {
                const int nc = (int)ctl.ncand;
                if (tid < nc) {
                    const unsigned long long mk = ckey[tid];
                    uint32_t wabove = 0;
                    for (int c = 0; c < nc; ++c)
                        if (ckey[c] > mk) wabove += clen[c];
                    if (wabove <= rem && wabove + clen[tid] > rem) ctl.thr = mk;
                }
                __syncthreads();
                thr = ctl.thr;
                break;
            }
            lo = ctl.lo;
            hi = ctl.hi;
            __syncthreads();
        }

        SKV_USTAMP(21);
        // 2d. ordered compaction (ascending ids + gathered token offsets)
        unsigned long long mine = 0;
        uint32_t kmin = 0xffffffffu;
        for (int i = c0; i < c1; ++i) {
            const int4 e = cand(i);
            if (all_fit || ukey64((uint32_t)e.x, e.y) > thr) {
                mine += (1ull << 32) | (uint32_t)e.w;
                kmin = min(kmin, (uint32_t)e.x);
            }
        }
        unsigned long long tot;
        const unsigned long long excl = block_incl_sum<unsigned long long>(mine, ws64, &tot) - mine;
        if (mine) {
            int pos = (int)(excl >> 32);
            int32_t toff = (int32_t)(excl & 0xffffffffull);
            for (int i = c0; i < c1; ++i) {
                const int4 e = cand(i);
                if (all_fit || ukey64((uint32_t)e.x, e.y) > thr) {
                    sel_tok[pos] = toff;
                    sel_src[pos] = e.z;
                    sel_id[pos] = e.y;
                    ++pos;
                    toff += e.w;
                }
            }
            atomicMin(&ctl.ks, kmin);
        }
        if (tid == 0) {
            const int count = (int)(tot >> 32);
            ctl.count = count;
            ctl.ntok = (int)(tot & 0xffffffffull);
            sel_tok[count] = ctl.ntok;
            ctl.kc = (uint32_t)(thr >> 32);
            ctl.kc_set = all_fit ? 0 : 1;
        }
        __syncthreads();
    }
    SKV_USTAMP(5);

    // ---------------------------------------------------------------- 3. gather + attend (D3 + D4)
    const int count = ctl.count, ntok = ctl.ntok;
    // NEXT-2 local segment: the tokens of the sentence being generated follow the selection in the
    // attended range (always attended, not charged to tau; generated rows are L + position)
    int hot0 = 0, nhot = 0;
    if (gen.Kg) {
        hot0 = gen.gstat[b * 4 + 1];
        nhot = gen.fixed + gen.gstat[b * 4 + 0] - hot0;  // the always-attended rows, then the hot sentence
    }
    const int natt = ntok + nhot;
    const int ntl = (natt + kTile - 1) / kTile;
    const int per = (ntl + kUC - 1) / kUC;
    const int tb = min(ntl, rank * per), te = min(ntl, tb + per);
    const int T0 = tb * kTile, T1 = min(natt, te * kTile);
    // first row index of the generated rows in the attention's row encoding: after the context rows
    // (device residency) or after the working-set rows (host residency)
    const int gbase = HOST ? hc.slots * kPage : gen.L;
    // Host residency (D3 host): the HBM working set is a page cache (pages of kPage context
    // rows); a page-table entry holds the page's slot and the mask of its rows already in HBM.  A
    // selected row is read from its slot if the row is there, else from the mapped host store.  When
    // a CTA meets such a miss it plans the cache for the whole selection (identically in every CTA:
    // ascending page / clock order): pages that are not resident get a slot whose page this selection
    // does not use (clock order from the hand), and the rows read from host are written through.
    // The plan is computed by the whole CTA in parallel (r02; the r01 version ran its page and slot
    // scans on one warp: ~9.5 us per plan): the selection's pages are marked in a page bitmap, their
    // ascending ranks come from one block scan over the bitmap words (rank(p) = word base + popcount
    // of the lower bits -- also the O(1) lookup of a row's plan entry), new pages are compacted by a
    // block scan, and the free slots in clock order from the hand by another.
    auto page_rank = [&](int p) -> int {
        return (int)pbase[p >> 5] + __popc(pbits[p >> 5] & ((1u << (p & 31)) - 1u));
    };
    auto cache_plan = [&]() {
        // the clock hand is loaded first and consumed late; the page-table entries of the selection are
        // read in ONE round, once the pages are ranked.  A slot is free iff no page of this selection
        // is in it (empty slots included); its owner is read only by the CTA that applies the plan.
        const int hand = hc.hand[unit];
        const int nwords = (hc.pages + 31) >> 5;
        for (int w = tid; w < nwords; w += kUT) pbits[w] = 0u;
        for (int j = tid; j < kMaxSlots / 32; j += kUT) inuse[j] = 0u;
        __syncthreads();
        SKV_USTAMP(26);
        for (int i = tid; i < count; i += kUT) {  // pages of the selection
            const int r0 = sel_src[i], r1 = r0 + (sel_tok[i + 1] - sel_tok[i]) - 1;
            if (HGEN && r0 >= hc.L) continue;  // a generated sentence (NEXT-2): not in the page cache
            for (int p = r0 / kPage; p <= r1 / kPage; ++p) atomicOr(&pbits[p >> 5], 1u << (p & 31));
        }
        if (ok && ctl.kc_set) {
            // band path: also give slots to the pages of the sentences just below the crossing point
            // (within w of it; no rows loaded): drift into them at the next steps then only fills rows in
            // (4w instead of w: more evictions of pages still in use later, +23 % host bytes, slower)
            const uint32_t kc = ctl.kc, klw = kc > (uint32_t)band_w ? kc - (uint32_t)band_w : 0u;
            const int* flg = reinterpret_cast<const int*>(gath + kUC * kUBandCap) + kUC * kUBandCap;
            for (int i = tid; i < ctl.base[kUC]; i += kUT) {
                const int4 e = gath[i];
                if (flg[i] || (uint32_t)e.x < klw || (uint32_t)e.x > kc || (HGEN && e.z >= hc.L)) continue;
                for (int p = e.z / kPage; p <= (e.z + e.w - 1) / kPage; ++p) atomicOr(&pbits[p >> 5], 1u << (p & 31));
            }
        }
        __syncthreads();
        SKV_USTAMP(27);
        uint32_t total;
        {   // word bases: exclusive prefix of the popcounts (thread t owns words [2t, 2t + 2))
            static_assert(2 * kUT >= kMaxPageWords, "two bitmap words per thread");
            uint32_t c[2], sum = 0;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int w = 2 * tid + k;
                c[k] = w < nwords ? __popc(pbits[w]) : 0u;
                sum += c[k];
            }
            uint32_t base = block_incl_sum<uint32_t>(sum, ws32, &total) - sum;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int w = 2 * tid + k;
                if (w < nwords) pbase[w] = base;
                base += c[k];
            }
            if (tid == 0) n_need_s = (int)min(total, (uint32_t)kNeedCap);
        }
        __syncthreads();
        const int n_need = n_need_s;
        for (int w = tid; w < nwords; w += kUT) {
            uint32_t m = pbits[w];
            int j = (int)pbase[w];
            while (m) {
                const int bit = __ffs(m) - 1;
                const int p = (w << 5) + bit;
                if (j < kNeedCap) {
                    need[j] = p;
                    rowbits[j] = 0u;
                } else {  // past the tracked pages (rare): still mark its slot as read by this step
                    const uint32_t e = (uint32_t)hc.pt[(size_t)unit * hc.pages + p];
                    if (e != kEmpty) atomicOr(&inuse[(e & 0xffffu) >> 5], 1u << (e & 31u));
                }
                ++j;
                m &= m - 1u;
            }
        }
        __syncthreads();
        for (int j = tid; j < n_need; j += kUT) {
            const uint32_t e = (uint32_t)hc.pt[(size_t)unit * hc.pages + need[j]];
            pslot[j] = e;
            slotof[j] = e == kEmpty ? -1 : (int)(e & 0xffffu);
            if (e != kEmpty) atomicOr(&inuse[(e & 0xffffu) >> 5], 1u << (e & 31u));
        }
        for (int i = tid; i < count; i += kUT) {  // the selected rows of every page
            const int r0 = sel_src[i], r1 = r0 + (sel_tok[i + 1] - sel_tok[i]) - 1;
            if (HGEN && r0 >= hc.L) continue;  // a generated sentence (NEXT-2): not in the page cache
            for (int p = r0 / kPage; p <= r1 / kPage; ++p) {
                const int j = page_rank(p);
                const int lo = max(r0, p * kPage) - p * kPage, hi = min(r1, p * kPage + kPage - 1) - p * kPage;
                if (j < kNeedCap) atomicOr(&rowbits[j], ((2u << hi) - 1u) & ~((1u << lo) - 1u));
            }
        }
        __syncthreads();
        SKV_USTAMP(28);
        // new pages (ascending) and free slots (clock order from the hand: empty, or holding a page
        // this selection does not use), both compacted by block scans (thread t owns 2 entries each)
        uint32_t nn = 0, nf = 0;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int j = 2 * tid + k;
            nn += (j < n_need && pslot[j] == kEmpty) ? 1u : 0u;
            int sl = hand + 2 * tid + k;
            sl = sl >= hc.slots ? sl - hc.slots : sl;
            nf += (2 * tid + k < hc.slots && !((inuse[sl >> 5] >> (sl & 31)) & 1u)) ? 1u : 0u;
        }
        // (the clock scan looks at the first 2 * kUT = 512 slots from the hand; the new pages are at most kNeedCap)
        static_assert(2 * kUT >= kNeedCap, "two entries per thread cover the new pages");
        uint32_t tot_new, tot_free;
        const uint32_t bn = block_incl_sum<uint32_t>(nn, ws32, &tot_new) - nn;
        const uint32_t bf = block_incl_sum<uint32_t>(nf, ws32, &tot_free) - nf;
        {
            uint32_t pn = bn, pf = bf;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int j = 2 * tid + k;
                if (j < n_need && pslot[j] == kEmpty) newj[pn++] = j;
                int sl = hand + 2 * tid + k;
                sl = sl >= hc.slots ? sl - hc.slots : sl;
                if (2 * tid + k < hc.slots && !((inuse[sl >> 5] >> (sl & 31)) & 1u)) {
                    if (pf < (uint32_t)kNeedCap) frees[pf] = sl;
                    ++pf;
                }
            }
        }
        __syncthreads();
        const int n_asg = (int)min(min(tot_new, tot_free), (uint32_t)kNeedCap);
        for (int k = tid; k < n_asg; k += kUT) {
            const int j = newj[k], sl = frees[k];
            slotof[j] = sl;
        }
        if (tid == 0) last_slot_s = n_asg > 0 ? frees[n_asg - 1] : -1;
        __syncthreads();
        SKV_USTAMP(29);
    };
    int my_miss = 0, my_new = 0;  // host rows read / of them in pages with no slot yet
    for (int t = T0 + tid; t < te * kTile; t += kUT) {
        int2 r = make_int2(kInvalid, -1);
        if (t < T1 && t >= ntok) {
            const int x = t - ntok;  // local segment: generated rows
            r.x = gbase + (x < gen.fixed ? x : hot0 + (x - gen.fixed));
        } else if (t < T1) {
            int lo2 = 0, hi2 = count - 1;  // largest i with sel_tok[i] <= t
            while (lo2 < hi2) {
                const int mid = (lo2 + hi2 + 1) >> 1;
                if (sel_tok[mid] <= t) lo2 = mid; else hi2 = mid - 1;
            }
            const int row = sel_src[lo2] + (t - sel_tok[lo2]);
            r.x = row;
            if (HGEN && row >= gen.L) {
                r.x = gbase + (row - gen.L);  // a generated sentence (NEXT-2): its rows are in HBM
            } else if constexpr (HOST) {
                const uint32_t e = (uint32_t)hc.pt[(size_t)unit * hc.pages + row / kPage];
                const int w = row % kPage;
                if (e != kEmpty && ((e >> (16 + w)) & 1u)) {
                    r.x = (int)(e & 0xffffu) * kPage + w;
                } else {
                    r.x = -(row + 1);
                    my_miss = 1;
                    if (e != kEmpty) r.y = (int)(e & 0xffffu) * kPage + w;  // its page has a slot: fill the row in
                    else my_new = 1;
                }
            }
        }
        rowtab[t - T0] = r;
    }
    const bool any_miss = __syncthreads_or(my_miss) != 0;  // (always false in device residency)
    // a plan is needed only for pages without a slot; rows missing from a page that has one are
    // written into it and published after barrier #2 (every CTA has done its lookups by then)
    const bool any_new = HOST && any_miss && __syncthreads_or(my_new) != 0;
#ifdef SKV_TRACE
    SKV_USTAMP(25);
    if (tid == 0 && unit * kUC + rank < 1024) g_unit_t[unit * kUC + rank][24] = any_miss ? 1 : 0;
#endif
    if (HOST && any_new) {
        cache_plan();
        // write-through targets of the rows read from host
        const int n_need = n_need_s;
        for (int t = T0 + tid; t < T1; t += kUT) {
            int2 r = rowtab[t - T0];
            if (r.x >= 0) continue;
            const int row = -(r.x + 1), p = row / kPage;
            const int j = page_rank(p);
            if (j < n_need && slotof[j] >= 0) {
                r.y = slotof[j] * kPage + row % kPage;
                rowtab[t - T0] = r;
            }
        }
        SKV_USTAMP(30);
        if (tid == 0) atomicMin(cluster.map_shared_rank(&ctl.miss_rank, 0), rank);  // lowest such rank updates the table
        __syncthreads();
    }
    SKV_USTAMP(6);
    // ---- stores of this step's state, spread over the CTAs (nothing waits on them) ----
    {
        const int sh = (count + kUC - 1) / kUC;  // selection entries written by this CTA
        int32_t* gids = sel.ids_of(cur, unit);
        int32_t* gtok = sel.tok_of(cur, unit);
        int32_t* gsrc = sel.src_of(cur, unit);
        for (int i = rank * sh + tid; i < min(count, (rank + 1) * sh); i += kUT) {
            gids[i] = sel_id[i];
            gtok[i] = sel_tok[i];
            gsrc[i] = sel_src[i];
            if (out_ids) out_ids[(size_t)unit * tau + i] = sid ? sid[(size_t)b * sid_stride + sel_id[i]] : sel_id[i];
        }
        if (out_ids) {
            const int pad = (tau - count + kUC - 1) / kUC;
            for (int i = count + rank * pad + tid; i < min(tau, count + (rank + 1) * pad); i += kUT)
                out_ids[(size_t)unit * tau + i] = -1;
        }
        if (rank == 0) {
            // deferred Eq. 2 state update: Sq += q_t, or reset after a boundary input (A11)
            const bool reset = ctl.reset != 0;
            for (int i = tid; i < GRP * D; i += kUT)
                Sq[((size_t)b * Hq + g * GRP) * D + i] = reset ? 0.0f : sqsum[i];
            if (tid == 0) {
                cnt[unit] = reset ? 0 : ctl.cnt0 + 1;
                gtok[count] = ntok;
                *sel.count_of(cur, unit) = count;
                if (out_count) out_count[unit] = count;
                if (out_tokens) out_tokens[unit] = ntok;
            }
        }
        if (rank == kUC - 1 && tid == 0) {
            // the next step's band: the crossing point and the lowest selected key, widened
            uint2 h = make_uint2(0u, 0xffffffffu);  // everything fits: the band is everything
            if (ctl.kc_set) {
                const uint32_t kc = ctl.kc, ks = ctl.ks, w = (uint32_t)band_w;
                const uint32_t wl = w << kBandLoShift;
                h.x = kc > wl ? kc - wl : 0u;
                h.y = ks < 0xffffffffu - w ? ks + w : 0xffffffffu;
            }
            hint[unit] = h;
        }
    }
    // the next kernel of the stream may start launching (it reads this step's state only after its
    // pdl_wait, i.e. after this grid has completed)
    pdl_trigger();
    auto attend = [&](auto miss_tag) {
        attend_phase<D, GRP, HOST, decltype(miss_tag)::value, !HOST || HGEN, MINB == 1>(
            rowtab, tb, te, T0, T1, q + ((size_t)b * Hq + g * GRP) * D,
            HOST ? hc.wsK + (size_t)unit * hc.slots * kPage * D : kv.K + (size_t)unit * kv.unit_stride * D,
            HOST ? hc.wsV + (size_t)unit * hc.slots * kPage * D : kv.V + (size_t)unit * kv.unit_stride * D,
            HOST ? hc.Kh + (size_t)unit * hc.L * D : nullptr, HOST ? hc.Vh + (size_t)unit * hc.L * D : nullptr,
            gen.Kg ? gen.Kg + (size_t)unit * gen.stride * D : nullptr,
            gen.Kg ? gen.Vg + (size_t)unit * gen.stride * D : nullptr, gbase, hc.ledger, scale_log2, msm);
    };
    if (HOST && any_miss) attend(std::true_type{});
    else attend(std::false_type{});
    SKV_USTAMP(7);
    cluster.sync();  // #2: CTA partials ready; every CTA has done its page-table lookups
    SKV_USTAMP(8);
    // host residency: the lowest rank that met a miss applies its plan (the same in every CTA that
    // computed one) after barrier #3 -- no other CTA recomputes it, and nobody waits for the update
    bool upd = false;
    if constexpr (HOST) {
        upd = any_new && *cluster.map_shared_rank(&ctl.miss_rank, 0) == rank;
        if (any_miss && !any_new) {  // no plan here: publish the rows this CTA wrote into resident pages
            int32_t* pt = hc.pt + (size_t)unit * hc.pages;
            for (int t = T0 + tid; t < T1; t += kUT) {
                const int2 r = rowtab[t - T0];
                if (r.x < 0 && r.y >= 0) {
                    const int row = -(r.x + 1);
                    atomicOr(&pt[row / kPage], (int32_t)(1u << (16 + row % kPage)));
                }
            }
        }
    }
    mma::merge_cluster<D, GRP, kUW, kUC>(cluster, msm, rank, out + ((size_t)b * Hq + g * GRP) * D, kUT, &peers,
                                         ((size_t)b * Hq + g * GRP) * D);
    cluster.sync();  // #3: remote reads done before any CTA of the cluster exits
    if (rank == 0 && tid == 0) {
        sel.parity[unit] = cur;
        if (peers.n) peers_arrive(peers);  // every CTA's slice is in every peer's buffer (8(e) fused gather)
    }
    if (HOST && upd) {
        // page-table update of this step's plan; all selected rows of a page with a slot are in it now.
        // (The next step reads the table after its programmatic-launch wait, i.e. after this grid.)
        const int n_need = n_need_s;
        int32_t* pt = hc.pt + (size_t)unit * hc.pages;
        for (int j = tid; j < n_need; j += kUT) {
            const int sl = slotof[j];
            if (sl < 0) continue;
            const uint32_t e = pslot[j];
            const uint32_t mask = (e == kEmpty ? 0u : (e >> 16)) | rowbits[j];
            if (e == kEmpty) {  // a new page: the slot's previous page (not in this selection) leaves
                const int old = hc.own[(size_t)unit * hc.slots + sl];
                if (old >= 0) pt[old] = (int32_t)kEmpty;
                hc.own[(size_t)unit * hc.slots + sl] = need[j];
            }
            pt[need[j]] = (int32_t)((uint32_t)sl | (mask << 16));
        }
        if (tid == 0 && last_slot_s >= 0) hc.hand[unit] = (last_slot_s + 1) % hc.slots;
    }
    SKV_USTAMP(9);
    SKV_LSTAMP(2);
}

size_t unit_smem_bytes(int d, int tau, int att) {
    (void)d;
    const size_t rows = (((size_t)att + kTile - 1) / kTile + kUC - 1) / kUC * kTile;  // attended tokens per CTA
    return (size_t)kUStages * kUTileBytes + sizeof(uint32_t) * kULocalCap + sizeof(int32_t) * (kULocalCap + 4) +
           sizeof(int4) * (kUOwnCap + kUBandCap) + sizeof(int32_t) * ((3 * (size_t)tau + 5) / 4 * 4) + sizeof(int2) * rows;
}

int unit_page_tokens() { return kPage; }

bool unit_supported(int d, int grp, int Smax, int tau, int slots, int pages, int local_att) {
    return (d == 64 || d == 128) && grp <= 8 && Smax <= kUC * kULocalCap &&
           unit_smem_bytes(d, tau, tau + local_att) <= 200 * 1024 &&
           slots <= kMaxSlots && pages <= kMaxPageWords * 32;
}

size_t unit_cand_entries(int units) { return (size_t)units * kUC * kULocalCap; }


static int trace_counter = 0;  // launch index for the trace build's per-launch stamps

template <int D, int GRP, bool HOST, bool HGEN, int MINB>
static cudaError_t launch_unit_t(const UnitArgs& a, cudaStream_t st) {
    const size_t smem = unit_smem_bytes(D, a.sel.tau, a.sel.tau + (a.gen.Kg ? a.gen.max_att : 0));
    cudaError_t e = ensure_smem((const void*)unit_step_kernel<D, GRP, HOST, HGEN, MINB>, smem);
    if (e != cudaSuccess) return e;
    const float scale_log2 = (float)(1.0 / sqrt((double)D) * 1.4426950408889634);
    return launch_pdl_if(a.pdl, unit_step_kernel<D, GRP, HOST, HGEN, MINB>, dim3(kUC, a.G, a.B), dim3(kUT), smem, st,
                      a.q, a.input_token,
                      a.bset, a.nb, a.Sq, a.cnt, a.E, a.S, a.off, a.off_stride, a.G, a.Smax, a.scores, a.sel, a.kv, a.hc,
                      a.cand, a.hint, a.band_w, a.out, a.out_ids,
                      a.out_count, a.out_tokens, a.sid, a.sid_stride, a.qmode, a.gen, a.peers, scale_log2,
                      trace_counter++);
}

// Two CTAs per SM fit the selection's shared memory (the kernel's static + dynamic + the per-CTA
// reservation, twice, within the SM's): then the kernel keeps <= 128 registers per thread (two
// CTAs' worth); else the instantiation with launch bounds (256, 1) may use the SM's registers for
// two attention tiles in flight per warp.
template <int D, int GRP, bool HOST, bool HGEN>
static bool unit_two_per_sm(size_t smem) {
    static const size_t fixed = [] {
        cudaFuncAttributes fa{};
        int dev = 0, resv = 0;
        cudaGetDevice(&dev);
        cudaFuncGetAttributes(&fa, (const void*)unit_step_kernel<D, GRP, HOST, HGEN, 2>);
        cudaDeviceGetAttribute(&resv, cudaDevAttrReservedSharedMemoryPerBlock, dev);
        return fa.sharedSizeBytes + (size_t)resv;
    }();
    static const size_t per_sm = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        return (size_t)v;
    }();
    return 2 * (smem + fixed) <= per_sm;
}

cudaError_t launch_unit(const UnitArgs& a, int grp, int d, cudaStream_t st) {
    const bool host = a.hc.Kh != nullptr;
    const size_t smem = unit_smem_bytes(d, a.sel.tau, a.sel.tau + (a.gen.Kg ? a.gen.max_att : 0));
#define SKV_UN2(DV, GV, H, HG)                                                                    \
    return unit_two_per_sm<DV, GV, H, HG>(smem) ? launch_unit_t<DV, GV, H, HG, 2>(a, st)        \
                                                : launch_unit_t<DV, GV, H, HG, 1>(a, st)
#define SKV_UN(DV, GV)                                   \
    if (!host) SKV_UN2(DV, GV, false, false);            \
    else if (a.gen.Kg) SKV_UN2(DV, GV, true, true);      \
    else SKV_UN2(DV, GV, true, false)
    if (d == 128) {
        switch (grp) {
            case 1: SKV_UN(128, 1);
            case 2: SKV_UN(128, 2);
            case 4: SKV_UN(128, 4);
            case 8: SKV_UN(128, 8);
        }
    } else {
        switch (grp) {
            case 1: SKV_UN(64, 1);
            case 2: SKV_UN(64, 2);
            case 4: SKV_UN(64, 4);
            case 8: SKV_UN(64, 8);
        }
    }
#undef SKV_UN
#undef SKV_UN2
    return cudaErrorInvalidValue;
}

}  // namespace skv
