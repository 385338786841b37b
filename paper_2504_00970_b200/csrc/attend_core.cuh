// attend_core.cuh -- D3 (bulk-copy gather of the selected sentences' K/V) + D4 (Eq. 3 attention)
// body shared by the attend kernel and the fused select+attend kernel.  See decode_attend.cu.
#pragma once
#include <cooperative_groups.h>

#include "device_util.cuh"
#include "skv_internal.cuh"

namespace skv {
namespace cg = cooperative_groups;

constexpr int kAttC = 64;         // tokens per chunk
constexpr int kAttThreads = 256;  // 8 warps
constexpr int kAttWarps = kAttThreads / 32;
constexpr int kCL = 8;            // CTAs per cluster (one cluster per (b, g) unit)
constexpr int kStages = 2;


template <int D, int GRP>
struct AttSmem {
    alignas(128) __nv_bfloat16 K[kStages][kAttC * D];  // reused as the cross-warp merge buffer
    alignas(128) __nv_bfloat16 V[kStages][kAttC * D];
    float p[kAttWarps][GRP][kAttC / kAttWarps];  // per-warp probabilities of the current chunk
    float mw[kAttWarps][GRP], lw[kAttWarps][GRP], sw[kAttWarps][GRP];  // per-warp running max / sum / rescale
    float m[GRP], l[GRP];                        // CTA partial (cluster merge reads it)
    alignas(16) float o[GRP * D];
    uint64_t bar[kStages];
    uint32_t done[kStages];                      // warps finished with the stage's current chunk
};

// Host residency (D3, "loaded from CPU back to the GPU memory"): where this unit's rows come
// from and go to.  A selected sentence that was also selected at the previous step is re-read from
// the previous working-set slot in HBM (src < 0 encodes row -(src+1) of that slot); the others are
// read from the mapped pinned host store over PCIe (src >= 0 = context row).  Every staged chunk is
// written through to the current slot, which becomes the next step's previous slot.
struct HostWs {
    const __nv_bfloat16* prevK;
    const __nv_bfloat16* prevV;
    __nv_bfloat16* curK;
    __nv_bfloat16* curV;
    unsigned long long* ledger;  // host bytes fetched (cumulative)
};

__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Issues the bulk copies of gathered chunk `c` (tokens [c*C, c*C+nc)) into stage `s`.  Called by
// one whole warp.  Selected sentence i occupies gathered tokens [tok[i], tok[i+1]) and rows
// [src[i], src[i] + tok[i+1] - tok[i]) of the attended store (context K/V, or with HOST the host
// store / previous working-set slot, see HostWs); tok / src are the shared-memory copies of the
// selection.  Returns the host bytes this lane requested.
template <int D, int GRP, bool HOST>
__device__ __forceinline__ uint32_t issue_chunk(AttSmem<D, GRP>& sm, int s, int c, int nc, const int32_t* tok,
                                                const int32_t* srcs, int count, const __nv_bfloat16* Kh,
                                                const __nv_bfloat16* Vh, const HostWs& ws, int lane) {
    uint32_t host = 0;
    const int c0 = c * kAttC;
    if (lane == 0) mbar_arrive_expect_tx(&sm.bar[s], (uint32_t)(nc * D * 2 * 2));
    __syncwarp();
    // largest i with tok[i] <= c0
    int lo = 0, hi = count - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (tok[mid] <= c0) lo = mid; else hi = mid - 1;
    }
    for (int i = lo + lane; i < count; i += 32) {
        const int ts = tok[i];
        if (ts >= c0 + nc) break;
        const int te = tok[i + 1];
        const int ps = max(ts, c0), pe = min(te, c0 + nc);
        const uint32_t bytes = (uint32_t)((pe - ps) * D * 2);
        const int v = srcs[i];
        if (HOST && v < 0) {
            const size_t src = (size_t)(-(v + 1) + (ps - ts)) * D;
            bulk_g2s(&sm.K[s][(ps - c0) * D], ws.prevK + src, bytes, &sm.bar[s]);
            bulk_g2s(&sm.V[s][(ps - c0) * D], ws.prevV + src, bytes, &sm.bar[s]);
        } else {
            const size_t src = (size_t)(v + (ps - ts)) * D;
            bulk_g2s(&sm.K[s][(ps - c0) * D], Kh + src, bytes, &sm.bar[s]);
            bulk_g2s(&sm.V[s][(ps - c0) * D], Vh + src, bytes, &sm.bar[s]);
            if (HOST) host += 2 * bytes;
        }
    }
    return host;
}

__device__ __forceinline__ void unpack8x2(const uint4& v, float2* f) {
    f[0] = make_float2(bf16lo(v.x), bf16hi(v.x));
    f[1] = make_float2(bf16lo(v.y), bf16hi(v.y));
    f[2] = make_float2(bf16lo(v.z), bf16hi(v.z));
    f[3] = make_float2(bf16lo(v.w), bf16hi(v.w));
}

// The chunk loop, warp merge and cluster merge for one (b, g) unit, run by every CTA of the
// unit's cluster once the selection metadata (tok[0..count], srcs[0..count)) is in its shared
// memory, the stage barriers are initialised and mw/lw are reset.  Writes out[(b*Hq+g*GRP)*D ..].
template <int D, int GRP, bool HOST = false>
__device__ __forceinline__ void attend_body(AttSmem<D, GRP>& sm, const int32_t* tok, const int32_t* srcs, int count,
                                            const __nv_bfloat16* Kh, const __nv_bfloat16* Vh,
                                            const __nv_bfloat16* __restrict__ q, float* __restrict__ out, int b,
                                            int g, int G, float scale_log2, cg::cluster_group& cluster,
                                            const HostWs& ws = HostWs{}) {
    constexpr int C = kAttC;
    constexpr int NW = kAttWarps;
    constexpr int SL = D / 8;           // 16-byte slices per row
    constexpr int TPW = 32 / SL;        // tokens per warp-row step
    constexpr int TW = C / NW;          // tokens per warp per chunk (8)
    constexpr int KT = TW / TPW;        // tokens per thread per chunk
    constexpr int N = GRP * KT;         // partial dots per thread per chunk
    static_assert(NW * GRP * D * 4 <= kStages * C * D * 2, "cross-warp merge buffer must fit in K");
    static_assert(32 % TW == 0, "softmax lane groups");
    const int rank = (int)cluster.block_rank();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int Hq = G * GRP;
    const int ntok = tok[count];
    const int nchunk = (ntok + C - 1) / C;
    const int per = (nchunk + kCL - 1) / kCL;
    const int cbeg = min(nchunk, rank * per), cend = min(nchunk, cbeg + per);
    const int mine = cend - cbeg;
    uint32_t host_bytes = 0;
    if (warp == 0)
        for (int s = 0; s < kStages && s < mine; ++s) {
            const int c = cbeg + s;
            host_bytes += issue_chunk<D, GRP, HOST>(sm, s, c, min(C, ntok - c * C), tok, srcs, count, Kh, Vh, ws, lane);
        }

    SKV_TRACE_POINT(2);
    const int slice = lane % SL, tsub = lane / SL;
    float2 q2[GRP][4];
#pragma unroll
    for (int h = 0; h < GRP; ++h)
        unpack8x2(*reinterpret_cast<const uint4*>(q + ((size_t)b * Hq + g * GRP + h) * D + slice * 8), q2[h]);
    float2 acc[GRP][4];
#pragma unroll
    for (int h = 0; h < GRP; ++h)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[h][i] = make_float2(0.0f, 0.0f);

    for (int it = 0; it < mine; ++it) {
        const int s = it % kStages;
        const int c = cbeg + it;
        const int nc = min(C, ntok - c * C);
        mbar_wait(&sm.bar[s], (it / kStages) & 1);
        if (it < 8) SKV_TRACE_POINT(3 + 2 * it);

        // ---- scores: thread (slice, tsub): warp tokens tsub + TPW*k, heads 0..GRP-1 ----
        float v[N];
#pragma unroll
        for (int k = 0; k < KT; ++k) {
            const int t = warp * TW + tsub + TPW * k;
            float2 k2[4];
            unpack8x2(*reinterpret_cast<const uint4*>(&sm.K[s][t * D + slice * 8]), k2);
#pragma unroll
            for (int h = 0; h < GRP; ++h) {
                float2 a2 = __fmul2_rn(q2[h][0], k2[0]);
#pragma unroll
                for (int i = 1; i < 4; ++i) a2 = __ffma2_rn(q2[h][i], k2[i], a2);
                v[h * KT + k] = a2.x + a2.y;
            }
        }
        // transpose-reduce over the SL lanes of a token group
        int base = 0, n = N;
#pragma unroll
        for (int o2 = SL / 2; o2 >= 1; o2 >>= 1) {
            if (n > 1) {
                const bool up = (lane & o2) != 0;
#pragma unroll
                for (int i = 0; i < N / 2; ++i) {
                    if (i < n / 2) {
                        const float send = up ? v[i] : v[i + n / 2];
                        const float keep = up ? v[i + n / 2] : v[i];
                        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o2);
                    }
                }
                if (up) base += n / 2;
                n /= 2;
            } else {
                v[0] += __shfl_xor_sync(0xffffffffu, v[0], o2);
            }
        }
        // scores -> the warp's private slab p[warp][h][local token]
#pragma unroll
        for (int i = 0; i < N; ++i) {
            if (i < n) {
                const int idx = base + i;
                const int h = idx / KT, k = idx % KT;
                const int tl = tsub + TPW * k;
                sm.p[warp][h][tl] = (warp * TW + tl) < nc ? v[i] * scale_log2 : -INFINITY;
            }
        }
        __syncwarp();
        // ---- per-warp online softmax: lane group of TW lanes per head ----
#pragma unroll
        for (int r = 0; r < (GRP * TW + 31) / 32; ++r) {
            const int j = r * 32 + lane;
            const int h = j / TW, tl = j % TW;
            const bool on = h < GRP;
            const float sv = on ? sm.p[warp][h][tl] : -INFINITY;
            float mx = sv;
#pragma unroll
            for (int w = TW / 2; w >= 1; w >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, w));
            const float m_old = on ? sm.mw[warp][h] : -INFINITY;
            const float m_new = fmaxf(m_old, mx);
            const float mref = m_new == -INFINITY ? 0.0f : m_new;
            const float pv = exp2f(sv - mref);
            float sum = pv;
#pragma unroll
            for (int w = TW / 2; w >= 1; w >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, w);
            if (on) {
                sm.p[warp][h][tl] = pv;
                if (tl == 0) {
                    const float sc = exp2f(m_old - mref);
                    sm.sw[warp][h] = sc;
                    sm.lw[warp][h] = sm.lw[warp][h] * sc + sum;
                    sm.mw[warp][h] = m_new;
                }
            }
        }
        __syncwarp();

        // ---- PV with rescaled accumulators ----
#pragma unroll
        for (int h = 0; h < GRP; ++h) {
            const float sc = sm.sw[warp][h];
            const float2 sc2 = make_float2(sc, sc);
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[h][i] = __fmul2_rn(acc[h][i], sc2);
        }
#pragma unroll
        for (int k = 0; k < KT; ++k) {
            const int tl = tsub + TPW * k;
            if (warp * TW + tl < nc) {
                float2 v2[4];
                unpack8x2(*reinterpret_cast<const uint4*>(&sm.V[s][(warp * TW + tl) * D + slice * 8]), v2);
#pragma unroll
                for (int h = 0; h < GRP; ++h) {
                    const float pp = sm.p[warp][h][tl];
                    const float2 p2 = make_float2(pp, pp);
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc[h][i] = __ffma2_rn(p2, v2[i], acc[h][i]);
                }
            }
        }
        if (it < 8) SKV_TRACE_POINT(4 + 2 * it);
        // ---- release the stage; the last warp out refills it ----
        __syncwarp();
        uint32_t last = 0;
        if (lane == 0) last = (atomicAdd(&sm.done[s], 1u) == (uint32_t)(NW - 1)) ? 1u : 0u;
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
            if (lane == 0) sm.done[s] = 0u;
            if (HOST && lane == 0) {
                // write the staged rows through to the current working-set slot (gathered order)
                bulk_s2g(ws.curK + (size_t)c * C * D, &sm.K[s][0], (uint32_t)(nc * D * 2));
                bulk_s2g(ws.curV + (size_t)c * C * D, &sm.V[s][0], (uint32_t)(nc * D * 2));
                bulk_commit();
                bulk_wait_read();  // the stage may be refilled once the store has read it
            }
            __syncwarp();
            if (it + kStages < mine) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                const int cn = c + kStages;
                host_bytes += issue_chunk<D, GRP, HOST>(sm, s, cn, min(C, ntok - cn * C), tok, srcs, count, Kh, Vh,
                                                        ws, lane);
            }
        }
    }

    pdl_trigger();
    // ---- merge the warps: reduce acc over the token groups of a warp, then over warps ----
#pragma unroll
    for (int w = SL; w < 32; w <<= 1)
#pragma unroll
        for (int h = 0; h < GRP; ++h)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                acc[h][i].x += __shfl_xor_sync(0xffffffffu, acc[h][i].x, w);
                acc[h][i].y += __shfl_xor_sync(0xffffffffu, acc[h][i].y, w);
            }
    SKV_TRACE_POINT(20);
    if (HOST) {
        bulk_wait_all();  // write-through stores complete (no-op for threads that issued none)
        unsigned long long hb = host_bytes;
#pragma unroll
        for (int o2 = 16; o2 >= 1; o2 >>= 1) hb += __shfl_xor_sync(0xffffffffu, hb, o2);
        if (lane == 0 && hb) atomicAdd(ws.ledger, hb);
    }
    __syncthreads();  // every warp is done with the stages
    float* red = reinterpret_cast<float*>(&sm.K[0][0]);  // [warps][GRP][D]
    if (tsub == 0) {
#pragma unroll
        for (int h = 0; h < GRP; ++h) {
            float* dst = &red[(warp * GRP + h) * D + slice * 8];
            *reinterpret_cast<float4*>(dst) = make_float4(acc[h][0].x, acc[h][0].y, acc[h][1].x, acc[h][1].y);
            *reinterpret_cast<float4*>(dst + 4) = make_float4(acc[h][2].x, acc[h][2].y, acc[h][3].x, acc[h][3].y);
        }
    }
    __syncthreads();
    if (tid < GRP) {
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < NW; ++w) M = fmaxf(M, sm.mw[w][tid]);
        const float Mref = M == -INFINITY ? 0.0f : M;
        float l = 0.0f;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const float e = exp2f(sm.mw[w][tid] - Mref);
            sm.sw[w][tid] = e;
            l = fmaf(e, sm.lw[w][tid], l);
        }
        sm.m[tid] = M;
        sm.l[tid] = l;
    }
    __syncthreads();
    for (int idx = tid; idx < GRP * D; idx += kAttThreads) {
        const int h = idx / D;
        float a = 0.0f;
#pragma unroll
        for (int w = 0; w < NW; ++w) a = fmaf(sm.sw[w][h], red[(w * GRP) * D + idx], a);
        sm.o[idx] = a;
    }

    // ---- merge the kCL partials through distributed shared memory ----
    SKV_TRACE_POINT(21);
    cluster.sync();
    SKV_TRACE_POINT(22);
    {
        // CTA r merges output elements [r*E, (r+1)*E) of the GRP*D outputs
        constexpr int E = (GRP * D + kCL - 1) / kCL;
        const int e0 = rank * E;
        for (int idx = e0 + tid; idx < min(GRP * D, e0 + E); idx += kAttThreads) {
            const int h = idx / D;
            float mr[kCL], lr[kCL], orr[kCL];
#pragma unroll
            for (int r = 0; r < kCL; ++r) {
                AttSmem<D, GRP>* rs = cluster.map_shared_rank(&sm, r);
                mr[r] = rs->m[h];
                lr[r] = rs->l[h];
                orr[r] = rs->o[idx];
            }
            float M = mr[0];
#pragma unroll
            for (int r = 1; r < kCL; ++r) M = fmaxf(M, mr[r]);
            float num = 0.0f, den = 0.0f;
#pragma unroll
            for (int r = 0; r < kCL; ++r) {
                const float w = (lr[r] > 0.0f) ? exp2f(mr[r] - M) : 0.0f;
                den = fmaf(w, lr[r], den);
                num = fmaf(w, orr[r], num);
            }
            out[((size_t)b * Hq + g * GRP) * D + idx] = num / den;
        }
    }
    SKV_TRACE_POINT(23);
    cluster.sync();  // keep every CTA's shared memory alive until all merges have read it
    SKV_TRACE_POINT(24);
}

}  // namespace skv
