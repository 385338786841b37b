// decode_attend.cu -- D3 (gather of the selected sentences' K/V) + D4 (Eq. 3 restricted
// attention) on sm_100a.
//
// D3: "CPU pairs associated with the retrieved tokens are loaded ... back to the GPU memory"
//     (Sec. 4.2; Alg. 1 line 18).  Device residency: the selected
//     sentences are contiguous token runs of K/V in HBM; each run piece is staged into shared
//     memory by one bulk async copy (TMA engine, cp.async.bulk) completing on an mbarrier.
// D4: O = softmax(q K_tau^T / sqrt(d)) V_tau (Eq. 3; Alg. 1 line 19), with the
//     current token's query per query head (A16), fp32 accumulation, fp32 output (A18).
//
// Split-K flash-decode: grid (nsplit, G, B); split c covers gathered tokens [c*C, c*C+C) of the
// (b, g) unit's selection.  All grp query heads of the KV head are processed together (GQA:
// each K/V byte is read once for grp heads).  Per split: partial (m, l, o) in the log2 domain;
// the last split CTA to finish (atomic ticket) merges the partials -- no extra launch.
#include "device_util.cuh"
#include "skv_internal.cuh"

namespace skv {

constexpr int kAttC = 64;        // tokens per split
constexpr int kAttThreads = 128; // 4 warps

int attend_chunk_tokens(int) { return kAttC; }

template <int D, int GRP>
struct AttSmem {
    alignas(128) __nv_bfloat16 K[kAttC * D];  // reused as the cross-warp PV reduction buffer
    alignas(128) __nv_bfloat16 V[kAttC * D];
    float p[GRP][kAttC];
    float m[GRP], l[GRP];
    uint64_t barK, barV;
    int last;
};

template <int D, int GRP>
__global__ void __launch_bounds__(kAttThreads) attend_kernel(
    const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ K, const __nv_bfloat16* __restrict__ V,
    int G, int L, const int32_t* __restrict__ off, int off_stride, const int32_t* __restrict__ sel_ids,
    const int32_t* __restrict__ sel_tokoff, const int32_t* __restrict__ sel_count, int tau, int nsplit,
    float* __restrict__ o_part, float* __restrict__ ml_part, uint32_t* __restrict__ done, float* __restrict__ out,
    float scale_log2) {
    constexpr int C = kAttC;
    constexpr int SL = D / 8;           // 16-byte slices per row
    constexpr int TPW = 32 / SL;        // tokens per warp-row step
    constexpr int KT = (C / 4) / TPW;   // tokens per thread (4 warps x 16 tokens)
    constexpr int N = GRP * KT;         // partial dots per thread
    static_assert(4 * GRP * D * 4 <= 2 * C * D, "PV reduction buffer must fit in the K tile");
    __shared__ AttSmem<D, GRP> sm;

    const int split = blockIdx.x, g = blockIdx.y, b = blockIdx.z;
    const int unit = b * G + g;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int count = sel_count[unit];
    const int32_t* tokoff = sel_tokoff + (size_t)unit * (tau + 1);
    const int ntok = tokoff[count];
    const int c0 = split * C;
    if (c0 >= ntok) return;
    const int nc = min(C, ntok - c0);
    const int nact = (ntok + C - 1) / C;
    const int Hq = G * GRP;

    // ---- D3: stage the chunk's K and V rows with bulk async copies ----
    if (tid == 0) {
        mbar_init(&sm.barK, 1);
        mbar_init(&sm.barV, 1);
    }
    __syncthreads();
    if (warp == 0) {
        if (lane == 0) {
            mbar_arrive_expect_tx(&sm.barK, (uint32_t)(nc * D * 2));
            mbar_arrive_expect_tx(&sm.barV, (uint32_t)(nc * D * 2));
        }
        __syncwarp();
        const int32_t* ids = sel_ids + (size_t)unit * tau;
        const int32_t* o = off + (size_t)b * off_stride;
        // largest i with tokoff[i] <= c0
        int lo = 0, hi = count - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (tokoff[mid] <= c0) lo = mid; else hi = mid - 1;
        }
        const size_t head_base = (size_t)unit * L;
        for (int i = lo + lane; i < count; i += 32) {
            const int ts = tokoff[i];
            if (ts >= c0 + nc) break;
            const int te = tokoff[i + 1];
            const int ps = max(ts, c0), pe = min(te, c0 + nc);
            const size_t src_tok = head_base + o[ids[i]] + (ps - ts);
            const uint32_t bytes = (uint32_t)((pe - ps) * D * 2);
            bulk_g2s(&sm.K[(ps - c0) * D], K + src_tok * D, bytes, &sm.barK);
            bulk_g2s(&sm.V[(ps - c0) * D], V + src_tok * D, bytes, &sm.barV);
        }
    }

    // query rows of this KV head's group, this thread's 8-dim slice, in registers
    const int slice = lane % SL, tsub = lane / SL;
    float qr[GRP][8];
#pragma unroll
    for (int h = 0; h < GRP; ++h) {
        const uint4 v = *reinterpret_cast<const uint4*>(q + ((size_t)b * Hq + g * GRP + h) * D + slice * 8);
        unpack8(v, qr[h]);
    }

    // ---- QK^T: thread (slice, tsub) of warp w: tokens 16w + tsub + TPW*k ----
    mbar_wait(&sm.barK, 0);
    float v[N];
#pragma unroll
    for (int k = 0; k < KT; ++k) {
        const int t = warp * 16 + tsub + TPW * k;
        float kf[8];
        unpack8(*reinterpret_cast<const uint4*>(&sm.K[t * D + slice * 8]), kf);
#pragma unroll
        for (int h = 0; h < GRP; ++h) {
            float acc = qr[h][0] * kf[0];
#pragma unroll
            for (int i = 1; i < 8; ++i) acc = fmaf(qr[h][i], kf[i], acc);
            v[h * KT + k] = acc;
        }
    }
    // transpose-reduce over the SL lanes of a token group: each halving step keeps half of the
    // values and adds the partner's copy of the same (head, token) entries.
    int base = 0;
    int n = N;
#pragma unroll
    for (int o = SL / 2; o >= 1; o >>= 1) {
        if (n > 1) {
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < N / 2; ++i) {
                if (i < n / 2) {
                    const float send = up ? v[i] : v[i + n / 2];
                    const float keep = up ? v[i + n / 2] : v[i];
                    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
            }
            if (up) base += n / 2;
            n /= 2;
        } else {
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
        }
    }
    // lane now holds entries [base, base + n) of the (head, token) list (when N < SL several
    // lanes hold the same fully reduced entry and store the same value)
#pragma unroll
    for (int i = 0; i < N; ++i) {
        if (i < n) {
            const int idx = base + i;
            const int h = idx / KT, k = idx % KT;
            const int t = warp * 16 + tsub + TPW * k;
            sm.p[h][t] = t < nc ? v[i] * scale_log2 : -INFINITY;
        }
    }
    __syncthreads();

    // ---- chunk softmax per head (log2 domain) ----
    for (int h = warp; h < GRP; h += 4) {
        const float s0 = sm.p[h][lane], s1 = sm.p[h][lane + 32];
        float mx = fmaxf(s0, s1);
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const float p0 = exp2f(s0 - mx), p1 = exp2f(s1 - mx);
        float sum = p0 + p1;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        sm.p[h][lane] = p0;
        sm.p[h][lane + 32] = p1;
        if (lane == 0) {
            sm.m[h] = mx;
            sm.l[h] = sum;
        }
    }
    __syncthreads();

    // ---- PV: same thread -> (slice, tokens) map as QK ----
    mbar_wait(&sm.barV, 0);
    float acc[GRP][8];
#pragma unroll
    for (int h = 0; h < GRP; ++h)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[h][i] = 0.0f;
#pragma unroll
    for (int k = 0; k < KT; ++k) {
        const int t = warp * 16 + tsub + TPW * k;
        if (t < nc) {
            float vf[8];
            unpack8(*reinterpret_cast<const uint4*>(&sm.V[t * D + slice * 8]), vf);
#pragma unroll
            for (int h = 0; h < GRP; ++h) {
                const float p = sm.p[h][t];
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[h][i] = fmaf(p, vf[i], acc[h][i]);
            }
        }
    }
    // reduce over the token groups of the warp (lanes differing in bits >= log2(SL))
#pragma unroll
    for (int o = SL; o < 32; o <<= 1)
#pragma unroll
        for (int h = 0; h < GRP; ++h)
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[h][i] += __shfl_xor_sync(0xffffffffu, acc[h][i], o);
    float* red = reinterpret_cast<float*>(sm.K);  // [4][GRP][D]; K tile is no longer read
    if (tsub == 0) {
#pragma unroll
        for (int h = 0; h < GRP; ++h)
#pragma unroll
            for (int i = 0; i < 8; i += 4)
                *reinterpret_cast<float4*>(&red[(warp * GRP + h) * D + slice * 8 + i]) =
                    make_float4(acc[h][i], acc[h][i + 1], acc[h][i + 2], acc[h][i + 3]);
    }
    __syncthreads();

    if (nact == 1) {
        for (int idx = tid; idx < GRP * D; idx += kAttThreads) {
            const int h = idx / D, j = idx % D;
            const float s = red[(0 * GRP + h) * D + j] + red[(1 * GRP + h) * D + j] + red[(2 * GRP + h) * D + j] +
                            red[(3 * GRP + h) * D + j];
            out[((size_t)b * Hq + g * GRP + h) * D + j] = s / sm.l[h];
        }
        return;
    }

    // ---- write this split's partial, then the last split CTA merges ----
    float* op = o_part + ((size_t)unit * nsplit + split) * GRP * D;
    for (int idx = tid; idx < GRP * D; idx += kAttThreads) {
        const int h = idx / D, j = idx % D;
        op[idx] = red[(0 * GRP + h) * D + j] + red[(1 * GRP + h) * D + j] + red[(2 * GRP + h) * D + j] +
                  red[(3 * GRP + h) * D + j];
    }
    if (tid < GRP) {
        float* ml = ml_part + (((size_t)unit * nsplit + split) * GRP + tid) * 2;
        ml[0] = sm.m[tid];
        ml[1] = sm.l[tid];
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) sm.last = (atomicAdd(&done[unit], 1u) == (uint32_t)(nact - 1));
    __syncthreads();
    if (!sm.last) return;
    __threadfence();
    const float* op0 = o_part + (size_t)unit * nsplit * GRP * D;
    const float* ml0 = ml_part + (size_t)unit * nsplit * GRP * 2;
    for (int idx = tid; idx < GRP * D; idx += kAttThreads) {
        const int h = idx / D;
        float M = -INFINITY;
        for (int i = 0; i < nact; ++i) M = fmaxf(M, __ldcg(&ml0[(i * GRP + h) * 2]));
        float num = 0.0f, den = 0.0f;
        for (int i = 0; i < nact; ++i) {
            const float w = exp2f(__ldcg(&ml0[(i * GRP + h) * 2]) - M);
            den = fmaf(w, __ldcg(&ml0[(i * GRP + h) * 2 + 1]), den);
            num = fmaf(w, __ldcg(&op0[(size_t)i * GRP * D + idx]), num);
        }
        out[((size_t)b * Hq + g * GRP) * D + idx] = num / den;
    }
    if (tid == 0) done[unit] = 0u;
}

template <int D>
static cudaError_t launch_attend_d(int grp, dim3 grid, cudaStream_t st, const __nv_bfloat16* q,
                                   const __nv_bfloat16* K, const __nv_bfloat16* V, int G, int L, const int32_t* off,
                                   int off_stride, const int32_t* sel_ids, const int32_t* sel_tokoff,
                                   const int32_t* sel_count, int tau, int nsplit, float* o_part, float* ml_part,
                                   uint32_t* done, float* out, float scale_log2) {
#define SKV_ATT(GRPV)                                                                                         \
    attend_kernel<D, GRPV><<<grid, kAttThreads, 0, st>>>(q, K, V, G, L, off, off_stride, sel_ids, sel_tokoff, \
                                                         sel_count, tau, nsplit, o_part, ml_part, done, out,   \
                                                         scale_log2)
    switch (grp) {
        case 1: SKV_ATT(1); break;
        case 2: SKV_ATT(2); break;
        case 4: SKV_ATT(4); break;
        case 8: SKV_ATT(8); break;
        default: return cudaErrorInvalidValue;
    }
#undef SKV_ATT
    return cudaGetLastError();
}

cudaError_t launch_attend(const __nv_bfloat16* q, const __nv_bfloat16* K, const __nv_bfloat16* V, int B, int G,
                          int grp, int d, int L, const int32_t* off, int off_stride, const int32_t* sel_ids,
                          const int32_t* sel_tokoff, const int32_t* sel_count, int tau, int chunk, int nsplit,
                          float* o_part, float* ml_part, uint32_t* done, float* out, cudaStream_t st) {
    (void)chunk;
    dim3 grid(nsplit, G, B);
    const float scale_log2 = (float)(1.0 / sqrt((double)d) * 1.4426950408889634);
    if (d == 128)
        return launch_attend_d<128>(grp, grid, st, q, K, V, G, L, off, off_stride, sel_ids, sel_tokoff, sel_count,
                                    tau, nsplit, o_part, ml_part, done, out, scale_log2);
    return launch_attend_d<64>(grp, grid, st, q, K, V, G, L, off, off_stride, sel_ids, sel_tokoff, sel_count, tau,
                               nsplit, o_part, ml_part, done, out, scale_log2);
}

}  // namespace skv
