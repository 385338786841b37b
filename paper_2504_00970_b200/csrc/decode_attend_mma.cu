// decode_attend_mma.cu -- D3 (gather) + D4 (Eq. 3 attention) with tensor-core MMAs.
//
// Same contract and results as attend_kernel / attend_host_kernel (decode_attend.cu); the work
// per token is done by mma.sync.m16n8k16 (bf16 in, fp32 accumulate), see mma_attend.cuh.
//
// One cluster of kMCL CTAs per (b, g) unit; each CTA owns a contiguous range of 16-token tiles of
// the unit's gathered tokens and its 8 warps take tiles round-robin, each with its own online
// softmax; warps merge through shared memory, CTAs through distributed shared memory.
#include <cooperative_groups.h>

#include "device_util.cuh"
#include "mma_attend.cuh"
#include "skv_internal.cuh"

namespace cg = cooperative_groups;

namespace skv {
SKV_TRACE_DEFINE(mma)

namespace {

constexpr int kMT = 256;   // threads per CTA
constexpr int kMW = kMT / 32;
constexpr int kMCL = 8;    // CTAs per cluster
using mma::kTile;
using mma::kInvalid;
template <int D>
using MmaSmem = mma::MergeSmem<D, kMW>;

}  // namespace

// HOST == false: rows come from kv (device residency, rows = context tokens).
// HOST == true:  srcs[i] >= 0 -> host row (mapped pinned store), < 0 -> row -(src+1) of the
//                previous working-set slot; every loaded row is written through to the current slot.
//                Rows >= L are generated rows (NEXT-2, HBM): never in the working set.
template <int D, int GRP, bool HOST>
__global__ void __cluster_dims__(kMCL, 1, 1) __launch_bounds__(kMT, 2)
attend_mma_kernel(const __nv_bfloat16* __restrict__ q, KvSrc kv, const __nv_bfloat16* Khost,
                  const __nv_bfloat16* Vhost, int L, __nv_bfloat16* wsK, __nv_bfloat16* wsV, int G, SelBufs sel,
                  unsigned long long* __restrict__ ledger, QsState qs, float* __restrict__ out, GenSrc gen,
                  OutPeers peers, float scale_log2) {
    static_assert(GRP <= 8, "heads fill the N = 8 side");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    MmaSmem<D>& sm = *reinterpret_cast<MmaSmem<D>*>(smem_raw);
    const int tau = sel.tau;
    int32_t* tok = reinterpret_cast<int32_t*>(smem_raw + sizeof(MmaSmem<D>));  // [tau + 1]
    int32_t* srcs = tok + (tau + 1);                                          // [tau]
    int32_t* pids = srcs + tau;                                               // [tau]     (HOST)
    int32_t* ptok = pids + tau;                                               // [tau + 1] (HOST)
    int32_t* rowtab = HOST ? ptok + (tau + 1) : pids;                         // [tiles per CTA * 16]

    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int g = blockIdx.y, b = blockIdx.z;
    const int unit = b * G + g;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int gq = lane >> 2, cq = lane & 3;  // mma groupID / thread-in-group
    const int Hq = G * GRP;

    SKV_TRACE_POINT(0);
    pdl_wait();
    if (rank == 0) qs_update_unit(q, qs.input_token, qs.bset, qs.nb, qs.Sq, qs.cnt, b, g, G, GRP, D, tid, kMT);
    const int prev = sel.parity[unit], cur = prev ^ 1;
    const int count = *sel.count_of(cur, unit);
    SKV_TRACE_POINT(1);
    {
        const int32_t* gt = sel.tok_of(cur, unit);
        const int32_t* gs = sel.src_of(cur, unit);
        for (int i = tid; i <= count; i += kMT) {
            tok[i] = gt[i];
            if (i < count) srcs[i] = gs[i];
        }
    }
    if (HOST) {
        const int pcount = *sel.count_of(prev, unit);
        const int32_t* pi = sel.ids_of(prev, unit);
        const int32_t* pt = sel.tok_of(prev, unit);
        for (int i = tid; i <= pcount; i += kMT) {
            if (i < pcount) pids[i] = pi[i];
            ptok[i] = pt[i];
        }
        __syncthreads();
        const int32_t* gi = sel.ids_of(cur, unit);
        for (int i = tid; i < count; i += kMT) {
            const int id = gi[i];
            int lo = 0, hi = pcount;  // first index with pids >= id
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (pids[mid] < id) lo = mid + 1; else hi = mid;
            }
            if (lo < pcount && pids[lo] == id && srcs[i] < L) srcs[i] = -(ptok[lo] + 1);
        }
    }
    __syncthreads();
    SKV_TRACE_POINT(2);
    const int ntok = tok[count];
    // NEXT-2 local segment: the generated sentence's tokens follow the selection
    int hot0 = 0, nhot = 0;
    if (gen.Kg) {
        hot0 = gen.gstat[b * 4 + 1];
        nhot = gen.fixed + gen.gstat[b * 4 + 0] - hot0;  // the always-attended rows, then the hot sentence
    }
    const int natt = ntok + nhot;
    const int ntiles = (natt + kTile - 1) / kTile;
    const int per = (ntiles + kMCL - 1) / kMCL;
    const int tb = min(ntiles, rank * per), te = min(ntiles, tb + per);
    const int T0 = tb * kTile, T1 = min(natt, te * kTile);
    // row of every gathered token of this CTA (HOST: encoded as above)
    for (int t = T0 + tid; t < te * kTile; t += kMT) {
        int r = kInvalid;
        if (t < T1 && t >= ntok) {
            const int x = t - ntok;
            r = gen.L + (x < gen.fixed ? x : hot0 + (x - gen.fixed));
        } else if (t < T1) {
            int lo = 0, hi = count - 1;  // largest i with tok[i] <= t
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (tok[mid] <= t) lo = mid; else hi = mid - 1;
            }
            const int v = srcs[lo], off = t - tok[lo];
            r = (HOST && v < 0) ? v - off : v + off;  // -(row+1) - off == -((row+off)+1)
        }
        rowtab[t - T0] = r;
    }
    __syncthreads();
    SKV_TRACE_POINT(3);

    const size_t ubase = (size_t)unit * kv.unit_stride + (size_t)cur * kv.slot_stride;
    const __nv_bfloat16* Kd = kv.K + ubase * D;  // device residency rows
    const __nv_bfloat16* Vd = kv.V + ubase * D;
    const __nv_bfloat16* Kh = HOST ? Khost + (size_t)unit * L * D : nullptr;
    const __nv_bfloat16* Vh = HOST ? Vhost + (size_t)unit * L * D : nullptr;
    const __nv_bfloat16* Kp = HOST ? wsK + ((size_t)unit * 2 + prev) * tau * D : nullptr;
    const __nv_bfloat16* Vp = HOST ? wsV + ((size_t)unit * 2 + prev) * tau * D : nullptr;
    __nv_bfloat16* Kc = HOST ? wsK + ((size_t)unit * 2 + cur) * tau * D : nullptr;
    __nv_bfloat16* Vc = HOST ? wsV + ((size_t)unit * 2 + cur) * tau * D : nullptr;
    const __nv_bfloat16* Kgu = gen.Kg ? gen.Kg + (size_t)unit * gen.stride * D : nullptr;
    const __nv_bfloat16* Vgu = gen.Kg ? gen.Vg + (size_t)unit * gen.stride * D : nullptr;
    auto rowK = [&](int r) -> const __nv_bfloat16* {
        if (!HOST) return (gen.Kg && r >= gen.L) ? Kgu + (size_t)(r - gen.L) * D : Kd + (size_t)r * D;
        if (Kgu && r >= L) return Kgu + (size_t)(r - L) * D;  // generated row (gen.L == L)
        return r >= 0 ? Kh + (size_t)r * D : Kp + (size_t)(-(r + 1)) * D;
    };
    auto rowV = [&](int r) -> const __nv_bfloat16* {
        if (!HOST) return (gen.Kg && r >= gen.L) ? Vgu + (size_t)(r - gen.L) * D : Vd + (size_t)r * D;
        if (Vgu && r >= L) return Vgu + (size_t)(r - L) * D;
        return r >= 0 ? Vh + (size_t)r * D : Vp + (size_t)(-(r + 1)) * D;
    };

    uint4 qseg[D / 32];
    mma::load_q<D, GRP>(qseg, q + ((size_t)b * Hq + g * GRP) * D, lane);
    mma::WarpAcc<D> wacc;
    wacc.init();
    unsigned long long host_bytes = 0;

    for (int tile = tb + warp; tile < te; tile += kMW) {
        const int t0 = tile * kTile;
        // ---- D3: rows of this tile (K: tokens gq, gq+8; V: tokens 2cq, 2cq+1, 2cq+8, 2cq+9) ----
        const int rk0 = rowtab[t0 + gq - T0], rk1 = rowtab[t0 + gq + 8 - T0];
        int rv[4];
        const __nv_bfloat16* pv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            rv[k] = rowtab[t0 + 2 * cq + (k & 1) + 8 * (k >> 1) - T0];
            pv[k] = rv[k] != kInvalid ? rowV(rv[k]) : nullptr;
        }
        mma::TileRegs<D> tr;
        mma::load_tile<D>(tr, rk0 != kInvalid ? rowK(rk0) : nullptr, rk1 != kInvalid ? rowK(rk1) : nullptr, pv, lane);
        if (tile == tb) SKV_TRACE_POINT(4);
        mma::compute_tile<D, GRP>(wacc, tr, qseg, t0 + gq < T1, t0 + gq + 8 < T1, scale_log2, lane);
        if (tile == tb) SKV_TRACE_POINT(6);
        if (tile == tb + kMW) SKV_TRACE_POINT(7);
        if (HOST) {
            constexpr int NU = D / 32, NVP = D / 64;
            // write the tile's context rows through to the current working-set slot (gathered order;
            // generated rows stay in their HBM store)
#pragma unroll
            for (int u = 0; u < NU; ++u) {
                if (rk0 != kInvalid && rk0 < L) *reinterpret_cast<uint4*>(Kc + (size_t)(t0 + gq) * D + mma::kseg(cq, u)) = tr.kA[u];
                if (rk1 != kInvalid && rk1 < L) *reinterpret_cast<uint4*>(Kc + (size_t)(t0 + gq + 8) * D + mma::kseg(cq, u)) = tr.kB[u];
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int pp = 0; pp < NVP; ++pp)
                    if (rv[k] != kInvalid && rv[k] < L)
                        *reinterpret_cast<uint4*>(Vc + (size_t)(t0 + 2 * cq + (k & 1) + 8 * (k >> 1)) * D + 8 * gq + 64 * pp) =
                            tr.vv[k][pp];
            // host bytes: K rows (counted once per row by cq == 0 lanes) + V rows (gq == 0 lanes)
            if (cq == 0) host_bytes += (rk0 >= 0 && rk0 < L ? D * 2 : 0) + (rk1 >= 0 && rk1 < L ? D * 2 : 0);
            if (gq == 0)
#pragma unroll
                for (int k = 0; k < 4; ++k) host_bytes += (rv[k] >= 0 && rv[k] < L) ? D * 2 : 0;
        }
    }
    if (HOST) {
        unsigned long long hb = host_bytes;
#pragma unroll
        for (int o2 = 16; o2 >= 1; o2 >>= 1) hb += __shfl_xor_sync(0xffffffffu, hb, o2);
        if (lane == 0 && hb) atomicAdd(ledger, hb);
    }

    SKV_TRACE_POINT(8);
    // ---- merge the warps (shared memory), then the kMCL CTA partials (distributed shared memory) ----
    mma::merge_warps<D, GRP, kMW>(sm, wacc, kMT);
    pdl_trigger();
    SKV_TRACE_POINT(9);
    cluster.sync();
    SKV_TRACE_POINT(10);
    mma::merge_cluster<D, GRP, kMW, kMCL>(cluster, sm, rank, out + ((size_t)b * Hq + g * GRP) * D, kMT, &peers,
                                          ((size_t)b * Hq + g * GRP) * D);
    SKV_TRACE_POINT(11);
    cluster.sync();
    SKV_TRACE_POINT(12);
    if (rank == 0 && tid == 0) {
        sel.parity[unit] = cur;
        if (peers.n) peers_arrive(peers);
    }
}

template <int D, int GRP, bool HOST>
static cudaError_t launch_mma_t(dim3 grid, cudaStream_t st, const __nv_bfloat16* q, KvSrc kv,
                                const __nv_bfloat16* Kh, const __nv_bfloat16* Vh, int L, __nv_bfloat16* wsK,
                                __nv_bfloat16* wsV, int G, SelBufs sel, unsigned long long* ledger, QsState qs,
                                float* out, GenSrc gen, OutPeers peers, float scale_log2) {
    // metadata: tok[tau+1] + srcs[tau] (+ pids[tau] + ptok[tau+1]) + rowtab[per-CTA tokens]; the
    // NEXT-2 local segment adds up to tau attended tokens
    const size_t tiles = ((size_t)sel.tau + (gen.Kg ? gen.max_att : 0) + kTile - 1) / kTile;
    const size_t rows = ((tiles + kMCL - 1) / kMCL) * kTile;
    const size_t meta = (size_t)(2 * sel.tau + 1) + (HOST ? (size_t)(2 * sel.tau + 1) : 0) + rows;
    const size_t smem = sizeof(MmaSmem<D>) + sizeof(int32_t) * meta;
    cudaError_t e = ensure_smem((const void*)attend_mma_kernel<D, GRP, HOST>, smem);
    if (e != cudaSuccess) return e;
    return launch_pdl_if(false, attend_mma_kernel<D, GRP, HOST>, grid, dim3(kMT), smem, st, q, kv, Kh, Vh, L, wsK, wsV, G, sel,
                      ledger, qs, out, gen, peers, scale_log2);
}

cudaError_t launch_attend_mma(const __nv_bfloat16* q, KvSrc kv, const __nv_bfloat16* Kh, const __nv_bfloat16* Vh,
                              int L, __nv_bfloat16* wsK, __nv_bfloat16* wsV, bool host, int B, int G, int grp, int d,
                              SelBufs sel, unsigned long long* ledger, QsState qs, float* out, GenSrc gen,
                              OutPeers peers, cudaStream_t st) {
    dim3 grid(kMCL, G, B);
    const float scale_log2 = (float)(1.0 / sqrt((double)d) * 1.4426950408889634);
#define SKV_MM(DV, GV)                                                                                          \
    return host ? launch_mma_t<DV, GV, true>(grid, st, q, kv, Kh, Vh, L, wsK, wsV, G, sel, ledger, qs, out, gen, peers, scale_log2) \
                : launch_mma_t<DV, GV, false>(grid, st, q, kv, Kh, Vh, L, wsK, wsV, G, sel, ledger, qs, out, gen, peers, scale_log2)
    if (d == 128) {
        switch (grp) {
            case 1: SKV_MM(128, 1);
            case 2: SKV_MM(128, 2);
            case 4: SKV_MM(128, 4);
            case 8: SKV_MM(128, 8);
        }
    } else {
        switch (grp) {
            case 1: SKV_MM(64, 1);
            case 2: SKV_MM(64, 2);
            case 4: SKV_MM(64, 4);
            case 8: SKV_MM(64, 8);
        }
    }
#undef SKV_MM
    return cudaErrorInvalidValue;
}

}  // namespace skv
