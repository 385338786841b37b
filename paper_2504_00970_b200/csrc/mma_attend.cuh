// mma_attend.cuh -- the tensor-core body of D4 (Eq. 3 attention) over gathered rows,
// shared by attend_mma_kernel (decode_attend_mma.cu) and the fused per-unit step kernel
// (decode_unit.cu).
//
// Work per 16-token tile, one warp, mma.sync.m16n8k16 (bf16 in, fp32 accumulate):
//   QK^T:  S^T[t][h] = sum_d K[t][d] q[h][d]   A = 16 tokens x 16 d (K rows), B = 16 d x 8 heads (q)
//   PV:    O^T[j][h] = sum_t V[t][j] P[h][t]   A = 16 dims x 16 tokens (V), B = 16 tokens x 8 heads (P)
// Heads fill the N = 8 side (grp = 4 or 8 query heads per KV head), so nothing is padded to 16.
// Operands are loaded straight from global memory into fragment registers with coalesced 128-bit
// loads (no shared-memory staging, no bank conflicts on 256-byte rows): the reduction index d is
// permuted -- identically for K and q -- so that each lane reads contiguous 16-byte segments of a
// row; pairs of V tokens are interleaved with byte permutes.  P is split into bf16 hi + lo parts
// (two MMAs) so the PV products keep ~16 mantissa bits.  Each warp keeps its own online softmax
// (log2 domain); warps merge through shared memory, CTAs of a cluster through DSMEM.
#pragma once
#include <cooperative_groups.h>

#include "device_util.cuh"

namespace skv {

// SURVEY 8(e), the per-layer all-gather fused into the attention epilogue: device pointers (UVA,
// peer-accessible: torch symmetric memory on NVLink) to every rank's gather buffer, already offset to
// THIS rank's slot, and to every rank's arrival counter for the layer.
constexpr int kMaxPeers = 8;
struct OutPeers {
    float* out[kMaxPeers];
    unsigned int* flag[kMaxPeers];
    int n;
};

// The unit's outputs are in every peer's buffer: count the arrival at every peer (release, system scope).
__device__ __forceinline__ void peers_arrive(const OutPeers& p) {
    for (int i = 0; i < p.n; ++i)
        asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(p.flag[i]) : "memory");
}

namespace mma {

constexpr int kTile = 16;  // tokens per MMA tile
constexpr int kInvalid = INT32_MIN;

__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t w_of(const uint4& v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

// bf16 element e (0..7) of x and of y interleaved into one register: lo = x[e], hi = y[e]
__device__ __forceinline__ uint32_t pair_elem(const uint4& x, const uint4& y, int e) {
    return __byte_perm(w_of(x, e >> 1), w_of(y, e >> 1), (e & 1) ? 0x7632 : 0x5410);
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(lo)) |
           ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(hi)) << 16);
}

__device__ __forceinline__ uint4 ldg16(const __nv_bfloat16* p) { return *reinterpret_cast<const uint4*>(p); }

// Per-warp state of the online softmax over the tiles a warp processed.  Lane (gq, cq) (mma
// groupID / thread-in-group) holds heads 2cq, 2cq+1.
template <int D>
struct WarpAcc {
    static constexpr int NKS = D / 16;  // k-steps of QK (and m-tiles of PV)
    float m[2], l[2];
    float acc[NKS][4];
    __device__ __forceinline__ void init() {
        m[0] = m[1] = -INFINITY;
        l[0] = l[1] = 0.0f;
#pragma unroll
        for (int i = 0; i < NKS; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0f;
    }
};

// Reduction-index permutation of QK (the same for K and q): piece u (8 consecutive d) of lane
// (gq, cq) starts at d = (4u + cq) * 8, so one load instruction of the 4 lanes of a row reads 64
// contiguous bytes (whole 32-byte sectors -- over PCIe, rows read from mapped host memory, each
// sector crosses the link once).
__device__ __forceinline__ constexpr int kseg(int cq, int u) { return (4 * u + cq) * 8; }

// q as the B operand of QK: lane (gq, cq) holds head gq, pieces kseg(cq, u)
template <int D, int GRP>
__device__ __forceinline__ void load_q(uint4 (&qseg)[D / 32], const __nv_bfloat16* qh0, int lane) {
    const int gq = lane >> 2, cq = lane & 3;
#pragma unroll
    for (int u = 0; u < D / 32; ++u)
        qseg[u] = gq < GRP ? ldg16(qh0 + (size_t)gq * D + kseg(cq, u)) : make_uint4(0, 0, 0, 0);
}

// Registers of one tile: K rows of tokens gq, gq+8 and V rows of tokens 2cq, 2cq+1, 2cq+8, 2cq+9.
template <int D>
struct TileRegs {
    static constexpr int NU = D / 32, NVP = D / 64;
    uint4 kA[NU], kB[NU];
    uint4 vv[4][NVP];
};

// Issues the loads of tile rows.  rk0/rk1: K row pointers (nullptr = padding token); rv: V rows.
template <int D>
__device__ __forceinline__ void load_tile(TileRegs<D>& t, const __nv_bfloat16* rk0, const __nv_bfloat16* rk1,
                                          const __nv_bfloat16* const (&rv)[4], int lane) {
    const int gq = lane >> 2, cq = lane & 3;
#pragma unroll
    for (int u = 0; u < TileRegs<D>::NU; ++u) {
        t.kA[u] = rk0 ? ldg16(rk0 + kseg(cq, u)) : make_uint4(0, 0, 0, 0);
        t.kB[u] = rk1 ? ldg16(rk1 + kseg(cq, u)) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int p = 0; p < TileRegs<D>::NVP; ++p)
            t.vv[k][p] = rv[k] ? ldg16(rv[k] + 8 * gq + 64 * p) : make_uint4(0, 0, 0, 0);
}

// QK^T, online softmax and PV of one loaded tile.  v0 / v1: tokens gq / gq+8 of the tile are real.
template <int D, int GRP>
__device__ __forceinline__ void compute_tile(WarpAcc<D>& w, const TileRegs<D>& t, const uint4 (&qseg)[D / 32],
                                             bool v0, bool v1, float scale_log2, int lane) {
    constexpr int NKS = D / 16, NVP = D / 64;
    const int gq = lane >> 2, cq = lane & 3;
    float s[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int j = 0; j < NKS; ++j) {
        const int u = j >> 1, h = (j & 1) * 2;
        const uint32_t a[4] = {w_of(t.kA[u], h), w_of(t.kB[u], h), w_of(t.kA[u], h + 1), w_of(t.kB[u], h + 1)};
        mma_bf16(s, a, w_of(qseg[u], h), w_of(qseg[u], h + 1));
    }
    float p[4];
#pragma unroll
    for (int e = 0; e < 2; ++e) {  // head 2cq + e
        const bool hv = 2 * cq + e < GRP;
        const float sa = (hv && v0) ? s[e] * scale_log2 : -INFINITY;
        const float sb = (hv && v1) ? s[2 + e] * scale_log2 : -INFINITY;
        float mx = fmaxf(sa, sb);
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
        const float m_new = fmaxf(w.m[e], mx);
        const float mref = m_new == -INFINITY ? 0.0f : m_new;
        p[e] = exp2f(sa - mref);
        p[2 + e] = exp2f(sb - mref);
        float sum = p[e] + p[2 + e];
        sum += __shfl_xor_sync(0xffffffffu, sum, 4);
        sum += __shfl_xor_sync(0xffffffffu, sum, 8);
        sum += __shfl_xor_sync(0xffffffffu, sum, 16);
        const float sc = exp2f(w.m[e] - mref);
        w.l[e] = w.l[e] * sc + sum;
        w.m[e] = m_new;
#pragma unroll
        for (int i = 0; i < NKS; ++i) {
            w.acc[i][e] *= sc;
            w.acc[i][2 + e] *= sc;
        }
    }
    // P^T as the B operand of PV: lane (gq, cq) needs P[head gq][tokens 2cq, 2cq+1, 2cq+8, 2cq+9],
    // held by lanes X = 8cq + gq/2 (tokens 2cq, 2cq+8) and Y = X + 4 (tokens 2cq+1, 2cq+9)
    const int X = 8 * cq + (gq >> 1), Y = X + 4, sel0 = gq & 1;
    float px[4], py[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        px[k] = __shfl_sync(0xffffffffu, p[k], X);
        py[k] = __shfl_sync(0xffffffffu, p[k], Y);
    }
    const float p00 = sel0 ? px[1] : px[0];  // token 2cq
    const float p01 = sel0 ? py[1] : py[0];  // token 2cq+1
    const float p10 = sel0 ? px[3] : px[2];  // token 2cq+8
    const float p11 = sel0 ? py[3] : py[2];  // token 2cq+9
    const uint32_t bh0 = pack_bf16(p00, p01), bh1 = pack_bf16(p10, p11);
    const uint32_t bl0 = pack_bf16(p00 - bf16lo(bh0), p01 - bf16hi(bh0));
    const uint32_t bl1 = pack_bf16(p10 - bf16lo(bh1), p11 - bf16hi(bh1));
    // PV: m-tile i rows -> dims (D=128: 8r+i / 64+8r+i; D=64: 8r+2i / 8r+2i+1)
#pragma unroll
    for (int i = 0; i < NKS; ++i) {
        uint32_t a[4];
        if (D == 128) {
            a[0] = pair_elem(t.vv[0][0], t.vv[1][0], i);
            a[1] = pair_elem(t.vv[0][NVP - 1], t.vv[1][NVP - 1], i);
            a[2] = pair_elem(t.vv[2][0], t.vv[3][0], i);
            a[3] = pair_elem(t.vv[2][NVP - 1], t.vv[3][NVP - 1], i);
        } else {
            a[0] = pair_elem(t.vv[0][0], t.vv[1][0], 2 * i);
            a[1] = pair_elem(t.vv[0][0], t.vv[1][0], 2 * i + 1);
            a[2] = pair_elem(t.vv[2][0], t.vv[3][0], 2 * i);
            a[3] = pair_elem(t.vv[2][0], t.vv[3][0], 2 * i + 1);
        }
        mma_bf16(w.acc[i], a, bh0, bh1);
        mma_bf16(w.acc[i], a, bl0, bl1);
    }
}

// Shared-memory area of the CTA merge (warps -> CTA partial) and the cluster merge (DSMEM).
template <int D, int NW>
struct MergeSmem {
    float red[NW][8][D];  // per-warp partial outputs (8 heads x D), rescaled to the CTA max
    float mw[NW][8], lw[NW][8];
    float m[8], l[8];     // CTA partial (cluster merge reads it)
    float o[8 * D];
};

// Warps -> CTA partial (sm.m, sm.l, sm.o: unnormalised, relative to sm.m).  All threads call it.
template <int D, int GRP, int NW>
__device__ __forceinline__ void merge_warps(MergeSmem<D, NW>& sm, const WarpAcc<D>& w, int nthreads) {
    constexpr int NKS = D / 16;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int gq = lane >> 2, cq = lane & 3;
    if (gq == 0) {
        sm.mw[warp][2 * cq] = w.m[0];
        sm.mw[warp][2 * cq + 1] = w.m[1];
        sm.lw[warp][2 * cq] = w.l[0];
        sm.lw[warp][2 * cq + 1] = w.l[1];
    }
    __syncthreads();
    float wsc[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int h = 2 * cq + e;
        float M = -INFINITY;
#pragma unroll
        for (int x = 0; x < NW; ++x) M = fmaxf(M, sm.mw[x][h]);
        wsc[e] = (w.m[e] == -INFINITY) ? 0.0f : exp2f(w.m[e] - M);
    }
    if (2 * cq < GRP) {  // lanes holding real heads only
#pragma unroll
        for (int i = 0; i < NKS; ++i) {
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const int dim = (D == 128) ? (half ? 64 + 8 * gq + i : 8 * gq + i) : (8 * gq + 2 * i + half);
                sm.red[warp][2 * cq][dim] = w.acc[i][2 * half] * wsc[0];
                if (2 * cq + 1 < GRP) sm.red[warp][2 * cq + 1][dim] = w.acc[i][2 * half + 1] * wsc[1];
            }
        }
    }
    __syncthreads();
    if (tid < GRP) {
        float M = -INFINITY;
#pragma unroll
        for (int x = 0; x < NW; ++x) M = fmaxf(M, sm.mw[x][tid]);
        float l = 0.0f;
#pragma unroll
        for (int x = 0; x < NW; ++x)
            if (sm.mw[x][tid] != -INFINITY) l += exp2f(sm.mw[x][tid] - M) * sm.lw[x][tid];
        sm.m[tid] = M;
        sm.l[tid] = l;
    }
    for (int idx = tid; idx < GRP * D; idx += nthreads) {
        const int h = idx / D, dim = idx % D;
        float a = 0.0f;
#pragma unroll
        for (int x = 0; x < NW; ++x) a += sm.red[x][h][dim];
        sm.o[idx] = a;
    }
}

// CTA partials of the cluster -> O (fp32, normalised).  Call after a cluster barrier that follows
// merge_warps in every CTA; CTA `rank` writes its 1/NC share of the GRP x D outputs to `out`.
template <int D, int GRP, int NW, int NC>
__device__ __forceinline__ void merge_cluster(cooperative_groups::cluster_group& cluster, MergeSmem<D, NW>& sm,
                                              int rank, float* __restrict__ out, int nthreads,
                                              const OutPeers* peers = nullptr, size_t peer_off = 0) {
    constexpr int E = (GRP * D + NC - 1) / NC;
    const int e0 = rank * E;
    for (int idx = e0 + (int)threadIdx.x; idx < min(GRP * D, e0 + E); idx += nthreads) {
        const int h = idx / D;
        float mr[NC], lr[NC], orr[NC];
#pragma unroll
        for (int r = 0; r < NC; ++r) {
            MergeSmem<D, NW>* rs = cluster.map_shared_rank(&sm, r);
            mr[r] = rs->m[h];
            lr[r] = rs->l[h];
            orr[r] = rs->o[idx];
        }
        float M = mr[0];
#pragma unroll
        for (int r = 1; r < NC; ++r) M = fmaxf(M, mr[r]);
        float num = 0.0f, den = 0.0f;
#pragma unroll
        for (int r = 0; r < NC; ++r) {
            const float w = (lr[r] > 0.0f) ? exp2f(mr[r] - M) : 0.0f;
            den = fmaf(w, lr[r], den);
            num = fmaf(w, orr[r], num);
        }
        const float o = num / den;
        out[idx] = o;
        if (peers)  // multi-GPU: the same value straight into this rank's slot of every peer's gather buffer
            for (int p = 0; p < peers->n; ++p) peers->out[p][peer_off + idx] = o;
    }
    if (peers && peers->n) asm volatile("fence.acq_rel.sys;" ::: "memory");  // before the flag release
}

}  // namespace mma
}  // namespace skv
