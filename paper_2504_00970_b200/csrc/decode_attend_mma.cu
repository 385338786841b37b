// decode_attend_mma.cu -- D3 (gather) + D4 (Eq. 3 attention) with tensor-core MMAs.
//
// Same contract and results as attend_kernel / attend_host_kernel (decode_attend.cu); the work
// per token is done by mma.sync.m16n8k16 (bf16 in, fp32 accumulate) instead of fp32 FMA:
//   QK^T:  S^T[t][h] = sum_d K[t][d] q[h][d]   A = 16 tokens x 16 d (K rows), B = 16 d x 8 heads (q)
//   PV:    O^T[j][h] = sum_t V[t][j] P[h][t]   A = 16 dims x 16 tokens (V), B = 16 tokens x 8 heads (P)
// Heads fill the N = 8 side (grp = 4 or 8 query heads per KV head), so nothing is padded to 16.
// Operands are loaded straight from global memory into fragment registers with coalesced 128-bit
// loads (no shared-memory staging, hence no bank conflicts on 256-byte rows): the reduction index
// d is permuted -- identically for K and q -- so that each lane reads contiguous 16-byte segments
// of a row; V pairs of tokens are interleaved with byte permutes.  P is split into bf16 hi + lo
// parts (two MMAs) so the PV products keep ~16 mantissa bits (H7 in SURVEY).
//
// One cluster of kCL CTAs per (b, g) unit; each CTA owns a contiguous range of 16-token tiles of
// the unit's gathered tokens and its 8 warps take tiles round-robin, each with its own online
// softmax; warps merge through shared memory, CTAs through distributed shared memory.
#include <cooperative_groups.h>

#include "device_util.cuh"
#include "skv_internal.cuh"

namespace cg = cooperative_groups;

namespace skv {
SKV_TRACE_DEFINE(mma)

namespace {

constexpr int kMT = 256;   // threads per CTA
constexpr int kMW = kMT / 32;
constexpr int kMCL = 8;    // CTAs per cluster
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

template <int D>
struct MmaSmem {
    float red[kMW][8][D];        // per-warp partial outputs (8 heads x D), rescaled to the CTA max
    float mw[kMW][8], lw[kMW][8];
    float m[8], l[8];            // CTA partial (cluster merge reads it)
    float o[8 * D];
};

}  // namespace

// HOST == false: rows come from kv (device residency, rows = context tokens).
// HOST == true:  srcs[i] >= 0 -> host row (mapped pinned store), < 0 -> row -(src+1) of the
//                previous working-set slot; every loaded row is written through to the current slot.
template <int D, int GRP, bool HOST>
__global__ void __cluster_dims__(kMCL, 1, 1) __launch_bounds__(kMT, 2)
attend_mma_kernel(const __nv_bfloat16* __restrict__ q, KvSrc kv, const __nv_bfloat16* Khost,
                  const __nv_bfloat16* Vhost, int L, __nv_bfloat16* wsK, __nv_bfloat16* wsV, int G, SelBufs sel,
                  unsigned long long* __restrict__ ledger, QsState qs, float* __restrict__ out, float scale_log2) {
    constexpr int NKS = D / 16;   // k-steps of QK (and m-tiles of PV)
    constexpr int NU = D / 32;    // 16-byte K segments per lane per row
    constexpr int NVP = D / 64;   // 16-byte V segments per lane per token (D = 64: 1, D = 128: 2)
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
            if (lo < pcount && pids[lo] == id) srcs[i] = -(ptok[lo] + 1);
        }
    }
    __syncthreads();
    SKV_TRACE_POINT(2);
    const int ntok = tok[count];
    const int ntiles = (ntok + kTile - 1) / kTile;
    const int per = (ntiles + kMCL - 1) / kMCL;
    const int tb = min(ntiles, rank * per), te = min(ntiles, tb + per);
    const int T0 = tb * kTile, T1 = min(ntok, te * kTile);
    // row of every gathered token of this CTA (HOST: encoded as above)
    for (int t = T0 + tid; t < te * kTile; t += kMT) {
        int r = kInvalid;
        if (t < T1) {
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
    auto rowK = [&](int r) -> const __nv_bfloat16* {
        if (!HOST) return Kd + (size_t)r * D;
        return r >= 0 ? Kh + (size_t)r * D : Kp + (size_t)(-(r + 1)) * D;
    };
    auto rowV = [&](int r) -> const __nv_bfloat16* {
        if (!HOST) return Vd + (size_t)r * D;
        return r >= 0 ? Vh + (size_t)r * D : Vp + (size_t)(-(r + 1)) * D;
    };

    // q as the B operand of QK: lane (gq, cq) holds head gq, d-range [cq*D/4, (cq+1)*D/4)
    uint4 qseg[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u)
        qseg[u] = gq < GRP ? ldg16(q + ((size_t)b * Hq + g * GRP + gq) * D + cq * (D / 4) + 8 * u)
                           : make_uint4(0, 0, 0, 0);
    float m2[2] = {-INFINITY, -INFINITY}, l2[2] = {0.0f, 0.0f};  // heads 2cq, 2cq+1
    float acc[NKS][4];
#pragma unroll
    for (int i = 0; i < NKS; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0f;
    unsigned long long host_bytes = 0;

    for (int tile = tb + warp; tile < te; tile += kMW) {
        const int t0 = tile * kTile;
        // ---- D3: rows of this tile (K: tokens gq, gq+8; V: tokens 2cq, 2cq+1, 2cq+8, 2cq+9) ----
        const int rk0 = rowtab[t0 + gq - T0], rk1 = rowtab[t0 + gq + 8 - T0];
        uint4 kA[NU], kB[NU];
#pragma unroll
        for (int u = 0; u < NU; ++u) {
            kA[u] = rk0 != kInvalid ? ldg16(rowK(rk0) + cq * (D / 4) + 8 * u) : make_uint4(0, 0, 0, 0);
            kB[u] = rk1 != kInvalid ? ldg16(rowK(rk1) + cq * (D / 4) + 8 * u) : make_uint4(0, 0, 0, 0);
        }
        int rv[4];
        uint4 vv[4][NVP];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            rv[k] = rowtab[t0 + 2 * cq + (k & 1) + 8 * (k >> 1) - T0];
#pragma unroll
            for (int p = 0; p < NVP; ++p)
                vv[k][p] = rv[k] != kInvalid ? ldg16(rowV(rv[k]) + 8 * gq + 64 * p) : make_uint4(0, 0, 0, 0);
        }
        // ---- QK^T: S^T[16 tokens][8 heads] ----
        if (tile == tb) SKV_TRACE_POINT(4);
        float s[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int j = 0; j < NKS; ++j) {
            const int u = j >> 1, h = (j & 1) * 2;
            const uint32_t a[4] = {w_of(kA[u], h), w_of(kB[u], h), w_of(kA[u], h + 1), w_of(kB[u], h + 1)};
            mma_bf16(s, a, w_of(qseg[u], h), w_of(qseg[u], h + 1));
        }
        if (tile == tb) SKV_TRACE_POINT(5);
        // ---- per-warp online softmax (log2 domain); lane holds tokens gq, gq+8 x heads 2cq, 2cq+1 ----
        const bool v0 = t0 + gq < T1, v1 = t0 + gq + 8 < T1;
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
            const float m_new = fmaxf(m2[e], mx);
            const float mref = m_new == -INFINITY ? 0.0f : m_new;
            p[e] = exp2f(sa - mref);
            p[2 + e] = exp2f(sb - mref);
            float sum = p[e] + p[2 + e];
            sum += __shfl_xor_sync(0xffffffffu, sum, 4);
            sum += __shfl_xor_sync(0xffffffffu, sum, 8);
            sum += __shfl_xor_sync(0xffffffffu, sum, 16);
            const float sc = exp2f(m2[e] - mref);
            l2[e] = l2[e] * sc + sum;
            m2[e] = m_new;
#pragma unroll
            for (int i = 0; i < NKS; ++i) {
                acc[i][e] *= sc;
                acc[i][2 + e] *= sc;
            }
        }
        // ---- P^T as the B operand of PV: lane (gq, cq) needs P[head gq][tokens 2cq, 2cq+1, 2cq+8, 2cq+9],
        //      held by lanes X = 8cq + gq/2 (tokens 2cq, 2cq+8) and Y = X + 4 (tokens 2cq+1, 2cq+9) ----
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
        // ---- PV: m-tile i rows -> dims (D=128: 8r+i / 64+8r+i; D=64: 8r+2i / 8r+2i+1) ----
#pragma unroll
        for (int i = 0; i < NKS; ++i) {
            uint32_t a[4];
            if (D == 128) {
                a[0] = pair_elem(vv[0][0], vv[1][0], i);
                a[1] = pair_elem(vv[0][NVP - 1], vv[1][NVP - 1], i);
                a[2] = pair_elem(vv[2][0], vv[3][0], i);
                a[3] = pair_elem(vv[2][NVP - 1], vv[3][NVP - 1], i);
            } else {
                a[0] = pair_elem(vv[0][0], vv[1][0], 2 * i);
                a[1] = pair_elem(vv[0][0], vv[1][0], 2 * i + 1);
                a[2] = pair_elem(vv[2][0], vv[3][0], 2 * i);
                a[3] = pair_elem(vv[2][0], vv[3][0], 2 * i + 1);
            }
            mma_bf16(acc[i], a, bh0, bh1);
            mma_bf16(acc[i], a, bl0, bl1);
        }
        if (tile == tb) SKV_TRACE_POINT(6);
        if (tile == tb + kMW) SKV_TRACE_POINT(7);
        if (HOST) {
            // write the tile's rows through to the current working-set slot (gathered order)
#pragma unroll
            for (int u = 0; u < NU; ++u) {
                if (rk0 != kInvalid) *reinterpret_cast<uint4*>(Kc + (size_t)(t0 + gq) * D + cq * (D / 4) + 8 * u) = kA[u];
                if (rk1 != kInvalid) *reinterpret_cast<uint4*>(Kc + (size_t)(t0 + gq + 8) * D + cq * (D / 4) + 8 * u) = kB[u];
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int pp = 0; pp < NVP; ++pp)
                    if (rv[k] != kInvalid)
                        *reinterpret_cast<uint4*>(Vc + (size_t)(t0 + 2 * cq + (k & 1) + 8 * (k >> 1)) * D + 8 * gq + 64 * pp) =
                            vv[k][pp];
            // host bytes: K rows (counted once per row by cq == 0 lanes) + V rows (gq == 0 lanes)
            if (cq == 0) host_bytes += (rk0 >= 0 ? D * 2 : 0) + (rk1 >= 0 ? D * 2 : 0);
            if (gq == 0)
#pragma unroll
                for (int k = 0; k < 4; ++k) host_bytes += (rv[k] >= 0 && rv[k] != kInvalid) ? D * 2 : 0;
        }
    }
    if (HOST) {
        unsigned long long hb = host_bytes;
#pragma unroll
        for (int o2 = 16; o2 >= 1; o2 >>= 1) hb += __shfl_xor_sync(0xffffffffu, hb, o2);
        if (lane == 0 && hb) atomicAdd(ledger, hb);
    }

    SKV_TRACE_POINT(8);
    // ---- merge the warps: CTA max per head, rescaled partial outputs summed through smem ----
    if (gq == 0) {
        sm.mw[warp][2 * cq] = m2[0];
        sm.mw[warp][2 * cq + 1] = m2[1];
        sm.lw[warp][2 * cq] = l2[0];
        sm.lw[warp][2 * cq + 1] = l2[1];
    }
    __syncthreads();
    float wsc[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int h = 2 * cq + e;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kMW; ++w) M = fmaxf(M, sm.mw[w][h]);
        wsc[e] = (m2[e] == -INFINITY) ? 0.0f : exp2f(m2[e] - M);
    }
#pragma unroll
    for (int i = 0; i < NKS; ++i) {
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const int r = gq + 8 * half;
            const int dim = (D == 128) ? (half ? 64 + 8 * gq + i : 8 * gq + i) : (8 * gq + 2 * i + half);
            (void)r;
            sm.red[warp][2 * cq][dim] = acc[i][2 * half] * wsc[0];
            sm.red[warp][2 * cq + 1][dim] = acc[i][2 * half + 1] * wsc[1];
        }
    }
    __syncthreads();
    if (tid < GRP) {
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kMW; ++w) M = fmaxf(M, sm.mw[w][tid]);
        float l = 0.0f;
#pragma unroll
        for (int w = 0; w < kMW; ++w)
            if (sm.mw[w][tid] != -INFINITY) l += exp2f(sm.mw[w][tid] - M) * sm.lw[w][tid];
        sm.m[tid] = M;
        sm.l[tid] = l;
    }
    for (int idx = tid; idx < GRP * D; idx += kMT) {
        const int h = idx / D, dim = idx % D;
        float a = 0.0f;
#pragma unroll
        for (int w = 0; w < kMW; ++w) a += sm.red[w][h][dim];
        sm.o[idx] = a;
    }
    pdl_trigger();
    SKV_TRACE_POINT(9);
    // ---- merge the kMCL partials through distributed shared memory ----
    cluster.sync();
    SKV_TRACE_POINT(10);
    {
        constexpr int E = (GRP * D + kMCL - 1) / kMCL;
        const int e0 = rank * E;
        for (int idx = e0 + tid; idx < min(GRP * D, e0 + E); idx += kMT) {
            const int h = idx / D;
            float mr[kMCL], lr[kMCL], orr[kMCL];
#pragma unroll
            for (int r = 0; r < kMCL; ++r) {
                MmaSmem<D>* rs = cluster.map_shared_rank(&sm, r);
                mr[r] = rs->m[h];
                lr[r] = rs->l[h];
                orr[r] = rs->o[idx];
            }
            float M = mr[0];
#pragma unroll
            for (int r = 1; r < kMCL; ++r) M = fmaxf(M, mr[r]);
            float num = 0.0f, den = 0.0f;
#pragma unroll
            for (int r = 0; r < kMCL; ++r) {
                const float w = (lr[r] > 0.0f) ? exp2f(mr[r] - M) : 0.0f;
                den = fmaf(w, lr[r], den);
                num = fmaf(w, orr[r], num);
            }
            out[((size_t)b * Hq + g * GRP) * D + idx] = num / den;
        }
    }
    SKV_TRACE_POINT(11);
    cluster.sync();
    SKV_TRACE_POINT(12);
    if (rank == 0 && tid == 0) sel.parity[unit] = cur;
}

template <int D, int GRP, bool HOST>
static cudaError_t launch_mma_t(dim3 grid, cudaStream_t st, const __nv_bfloat16* q, KvSrc kv,
                                const __nv_bfloat16* Kh, const __nv_bfloat16* Vh, int L, __nv_bfloat16* wsK,
                                __nv_bfloat16* wsV, int G, SelBufs sel, unsigned long long* ledger, QsState qs,
                                float* out, float scale_log2) {
    // metadata: tok[tau+1] + srcs[tau] (+ pids[tau] + ptok[tau+1]) + rowtab[per-CTA tokens]
    const size_t tiles = ((size_t)sel.tau + kTile - 1) / kTile;
    const size_t rows = ((tiles + kMCL - 1) / kMCL) * kTile;
    const size_t meta = (size_t)(2 * sel.tau + 1) + (HOST ? (size_t)(2 * sel.tau + 1) : 0) + rows;
    const size_t smem = sizeof(MmaSmem<D>) + sizeof(int32_t) * meta;
    static size_t configured = 0;
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(attend_mma_kernel<D, GRP, HOST>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(attend_mma_kernel<D, GRP, HOST>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    return launch_pdl(attend_mma_kernel<D, GRP, HOST>, grid, dim3(kMT), smem, st, q, kv, Kh, Vh, L, wsK, wsV, G, sel,
                      ledger, qs, out, scale_log2);
}

bool mma_enabled() {
    static const bool on = [] {
        const char* e = getenv("SKV_ATTEND");
        return !(e && e[0] == 'f');  // SKV_ATTEND=fma selects the fp32-FMA attend kernels
    }();
    return on;
}

cudaError_t launch_attend_mma(const __nv_bfloat16* q, KvSrc kv, const __nv_bfloat16* Kh, const __nv_bfloat16* Vh,
                              int L, __nv_bfloat16* wsK, __nv_bfloat16* wsV, bool host, int B, int G, int grp, int d,
                              SelBufs sel, unsigned long long* ledger, QsState qs, float* out, cudaStream_t st) {
    dim3 grid(kMCL, G, B);
    const float scale_log2 = (float)(1.0 / sqrt((double)d) * 1.4426950408889634);
#define SKV_MM(DV, GV)                                                                                          \
    return host ? launch_mma_t<DV, GV, true>(grid, st, q, kv, Kh, Vh, L, wsK, wsV, G, sel, ledger, qs, out, scale_log2) \
                : launch_mma_t<DV, GV, false>(grid, st, q, kv, Kh, Vh, L, wsK, wsV, G, sel, ledger, qs, out, scale_log2)
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
