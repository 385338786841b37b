// retain.cu -- SURVEY 8(f) NEXT-1, importance-filtered retention at prefill (Sec. 4.1, P:393-410;
// Alg. 1 lines 4-7; global top-k, App. "Effect of Sentence Length").
//
//   alpha_j = sum over the N window queries w and all Hq heads h of softmax_j(q_{w,h} . k_j / sqrt(d))
//   over the causal prefix of w, for the candidates j < L - N (reading A21); keep the global top
//   floor(r * tau) tokens (ties -> lowest index); every sentence keeps its retained tokens (pool in
//   token order, reading A25 drops sentences with none); Eq. 1 then runs over the pool.
//
// The window attention is a real dense contraction -- per (sequence, KV head) unit the R = N * grp
// window rows (128 for N = 32 and Llama-8B's grp = 4) against L keys -- so it runs on the 5th-gen
// tensor cores: tcgen05.mma (bf16 in, fp32 accumulate in TMEM) fed by TMA tensor loads in a 4-stage
// ring, one elected thread issuing, four epilogue warps reading the accumulator with tcgen05.ld.
// Two passes because alpha needs every row's final softmax normaliser:
//   pass A (rows on the MMA's M side): per row, running max and sum of exp over a chunk of keys;
//          the chunks are combined by alpha_rowcombine_kernel (fixed order);
//   pass B (keys on M, rows on N): per key, sum over rows of exp(z - m_row) / l_row, the KV heads
//          of the sequence looped inside the CTA in ascending order, so alpha is summed in one
//          fixed order without atomics (bit-identical run to run).
// Both passes are bound by the exp2 of every (row, key) score (MUFU), not by HBM (each reads K once).
#include <cuda.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "device_util.cuh"
#include "skv_internal.cuh"
#include "umma.cuh"

namespace skv {
namespace {

constexpr int kKT = 128;             // keys per tile
constexpr int kStages = 2;           // K-tile ring (2 stages: two CTAs per SM, 8 epilogue warps)
constexpr int kHalf = 128 * 128;     // one TMA box: 128 rows x 64 bf16 (128 B, swizzled) = 16 KB
constexpr int kThreads = 192;        // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue
constexpr int kMaxTiles = 16;        // pass B: key tiles per CTA (alpha kept in shared memory)

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// 2^x on the SFU, flush-to-zero (x <= 0 here: results below 2^-126 are far below the tolerance)
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// mbarrier wait that traps (a launch error, not a hung GPU) if the pipeline ever stalls for seconds
__device__ __forceinline__ void wait_or_trap(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    for (long long spin = 0; !done; ++spin) {
        asm volatile(
            "{\n.reg .pred P1;\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
        if (spin > (1ll << 26)) __trap();
    }
}

// ---------------------------------------------------------------------------- pass A: row stats
template <int DH>
__global__ void __launch_bounds__(kThreads, 2)
alpha_rowstats_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK, int L, int N,
                      int grp, int G, int R, int nrb, int wbox, int chunk_tiles, float scale_log2,
                      float2* __restrict__ part) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    unsigned char* sQ = sm;                 // DH boxes: window rows of this row block
    unsigned char* sK = sm + DH * kHalf;    // kStages x DH boxes
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages], tfull[2], tempty[2], qbar;
    __shared__ uint32_t tmem_base;

    const int chunk = blockIdx.x, g = blockIdx.y / nrb, rb = blockIdx.y % nrb, b = blockIdx.z;
    const int nchunk = gridDim.x;
    const int t0 = chunk * chunk_tiles, t1 = min((L + kKT - 1) / kKT, t0 + chunk_tiles);
    const int nt = t1 - t0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        mbar_init(&qbar, 1);
    }
    if (warp == 1) umma::tmem_alloc(&tmem_base, 256);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tbase = tmem_base;

    if (warp == 0 && lane == 0) {
        // ---- TMA producer
        umma::tma_prefetch(&tmQ);
        umma::tma_prefetch(&tmK);
        mbar_arrive_expect_tx(&qbar, (uint32_t)(DH * grp * wbox * 128));
        for (int h = 0; h < DH; ++h) umma::tma_load_3d(sQ + h * kHalf, &tmQ, h * 64, g * grp, b * N + rb * wbox, &qbar);
        for (int i = 0; i < nt; ++i) {
            const int s = i % kStages;
            if (i >= kStages) wait_or_trap(&empty[s], ((i / kStages) - 1) & 1);
            mbar_arrive_expect_tx(&full[s], (uint32_t)(DH * kHalf));
            for (int h = 0; h < DH; ++h)
                umma::tma_load_2d(sK + (s * DH + h) * kHalf, &tmK, h * 64, (b * G + g) * L + (t0 + i) * kKT, &full[s]);
        }
    } else if (warp == 1 && lane == 0) {
        // ---- MMA issuer: D[row][key] = Q[row] . K[key] (M = 128 rows, N = 128 keys, K = d)
        constexpr uint32_t idesc = umma::idesc_bf16_f32(128, kKT);
        wait_or_trap(&qbar, 0);
        for (int i = 0; i < nt; ++i) {
            const int s = i % kStages, acc = i & 1;
            wait_or_trap(&full[s], (i / kStages) & 1);
            if (i >= 2) wait_or_trap(&tempty[acc], ((i >> 1) - 1) & 1);
            umma::fence_after();
#pragma unroll
            for (int kk = 0; kk < DH * 4; ++kk) {
                const int h = kk >> 2, k4 = kk & 3;
                const uint64_t a = umma::desc_k128(smem_addr(sQ + h * kHalf) + k4 * 32);
                const uint64_t bd = umma::desc_k128(smem_addr(sK + (s * DH + h) * kHalf) + k4 * 32);
                umma::mma_bf16(tbase + acc * kKT, a, bd, idesc, kk > 0 ? 1u : 0u);
            }
            umma::commit(&empty[s]);
            umma::commit(&tfull[acc]);
        }
    } else if (warp >= 2) {
        // ---- epilogue: thread = window row; running max / sum of exp2 over the causal prefix
        const int quarter = warp & 3, row = quarter * 32 + lane;
        const int rg = rb * 128 + row;
        const int w = rg / grp;
        const int p = L - N + w;  // the row's window token sees keys 0..p
        float m = -INFINITY, l = 0.0f;
        for (int i = 0; i < nt; ++i) {
            const int acc = i & 1;
            wait_or_trap(&tfull[acc], (i >> 1) & 1);
            umma::fence_after();
            const int jb = (t0 + i) * kKT;
            const bool masked = jb + kKT - 1 > L - N;  // only tiles reaching the window need the causal mask
#pragma unroll 1
            for (int c4 = 0; c4 < 4; ++c4) {
                float v[32];
                umma::ld32(tbase + ((uint32_t)(quarter * 32) << 16) + acc * kKT + c4 * 32, v);
                float cm = -INFINITY;
                if (masked) {
#pragma unroll
                    for (int c = 0; c < 32; ++c) v[c] = (jb + c4 * 32 + c <= p) ? v[c] * scale_log2 : -INFINITY;
                } else {
#pragma unroll
                    for (int c = 0; c < 32; ++c) v[c] *= scale_log2;
                }
#pragma unroll
                for (int c = 0; c < 32; ++c) cm = fmaxf(cm, v[c]);
                if (cm == -INFINITY) continue;
                if (cm > m) {
                    l *= ex2(m - cm);
                    m = cm;
                }
                float s4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
                for (int c = 0; c < 32; ++c) s4[c & 3] += ex2(v[c] - m);
                l += (s4[0] + s4[1]) + (s4[2] + s4[3]);
            }
            umma::fence_before();
            __syncwarp();
            if (lane == 0) umma::mbar_arrive(&tempty[acc]);
        }
        if (rg < R && row < grp * wbox)
            part[((size_t)((b * G + g) * nrb + rb) * nchunk + chunk) * 128 + row] = make_float2(m, l);
    }
    __syncthreads();
    if (warp == 1) {
        umma::fence_after();
        umma::tmem_free(tbase, 256);
    }
}

// (m, l) of every window row: combine the chunks of pass A in ascending chunk order.
__global__ void alpha_rowcombine_kernel(const float2* __restrict__ part, int G, int R, int nrb, int nchunk,
                                        float2* __restrict__ stats) {
    const int g = blockIdx.x, b = blockIdx.y;
    for (int r = threadIdx.x; r < R; r += blockDim.x) {
        const float2* pp = part + ((size_t)((b * G + g) * nrb + r / 128) * nchunk) * 128 + (r % 128);
        float m = -INFINITY;
        for (int c = 0; c < nchunk; ++c) m = fmaxf(m, pp[(size_t)c * 128].x);
        float l = 0.0f;
        for (int c = 0; c < nchunk; ++c) {
            const float2 v = pp[(size_t)c * 128];
            if (v.x != -INFINITY) l += v.y * exp2f(v.x - m);
        }
        stats[(size_t)(b * G + g) * R + r] = make_float2(m, 1.0f / l);
    }
}

// ---------------------------------------------------------------------------- pass B: alpha
template <int DH>
__global__ void __launch_bounds__(kThreads, 2)
alpha_colsum_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK, int L, int N,
                    int grp, int G, int R, int Lc, int tiles_per_cta, int qhalf, float scale_log2,
                    const float2* __restrict__ stats, float* __restrict__ alpha) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    unsigned char* sQ = sm;                     // DH halves of R rows, qhalf bytes apart
    unsigned char* sK = sm + DH * qhalf;        // kStages x DH boxes
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages], tfull[2], tempty[2], qfull, qempty;
    __shared__ uint32_t tmem_base;
    __shared__ __align__(16) float2 sstat[2][256];
    __shared__ float salpha[kMaxTiles][kKT];

    const int b = blockIdx.y;
    const int ntc = (Lc + kKT - 1) / kKT;
    const int t0 = blockIdx.x * tiles_per_cta, t1 = min(ntc, t0 + tiles_per_cta);
    const int nt = t1 - t0;
    const int rc = (R + 31) / 32 * 32;          // TMEM columns per accumulator
    const uint32_t ncols = rc * 2 <= 64 ? 64 : rc * 2 <= 128 ? 128 : rc * 2 <= 256 ? 256 : 512;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        mbar_init(&qfull, 1);
        mbar_init(&qempty, 1);
    }
    if (warp == 1) umma::tmem_alloc(&tmem_base, ncols);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tbase = tmem_base;

    if (warp == 0 && lane == 0) {
        umma::tma_prefetch(&tmQ);
        umma::tma_prefetch(&tmK);
        for (int g = 0; g < G; ++g) {
            if (g > 0) wait_or_trap(&qempty, (g - 1) & 1);
            mbar_arrive_expect_tx(&qfull, (uint32_t)(DH * R * 128));
            for (int h = 0; h < DH; ++h) umma::tma_load_3d(sQ + h * qhalf, &tmQ, h * 64, g * grp, b * N, &qfull);
            for (int i = 0; i < nt; ++i) {
                const int it = g * nt + i, s = it % kStages;
                if (it >= kStages) wait_or_trap(&empty[s], ((it / kStages) - 1) & 1);
                mbar_arrive_expect_tx(&full[s], (uint32_t)(DH * kHalf));
                for (int h = 0; h < DH; ++h)
                    umma::tma_load_2d(sK + (s * DH + h) * kHalf, &tmK, h * 64, (b * G + g) * L + (t0 + i) * kKT, &full[s]);
            }
        }
    } else if (warp == 1 && lane == 0) {
        // D[key][row] = K[key] . Q[row] (M = 128 keys, N = R rows)
        const uint32_t idesc = umma::idesc_bf16_f32(128, R);
        for (int g = 0; g < G; ++g) {
            wait_or_trap(&qfull, g & 1);
            for (int i = 0; i < nt; ++i) {
                const int it = g * nt + i, s = it % kStages, acc = it & 1;
                wait_or_trap(&full[s], (it / kStages) & 1);
                if (it >= 2) wait_or_trap(&tempty[acc], ((it >> 1) - 1) & 1);
                umma::fence_after();
#pragma unroll
                for (int kk = 0; kk < DH * 4; ++kk) {
                    const int h = kk >> 2, k4 = kk & 3;
                    const uint64_t a = umma::desc_k128(smem_addr(sK + (s * DH + h) * kHalf) + k4 * 32);
                    const uint64_t bq = umma::desc_k128(smem_addr(sQ + h * qhalf) + k4 * 32);
                    umma::mma_bf16(tbase + acc * rc, a, bq, idesc, kk > 0 ? 1u : 0u);
                }
                umma::commit(&empty[s]);
                umma::commit(&tfull[acc]);
            }
            umma::commit(&qempty);  // this head's Q may be overwritten once its MMAs are done
        }
    } else if (warp >= 2) {
        // thread = key of the tile: alpha_j += sum over rows (ascending) of exp2(z - m) / l
        const int et = threadIdx.x - 64, quarter = warp & 3, row = quarter * 32 + lane;
        for (int g = 0; g < G; ++g) {
            // rows R..rc-1 (TMEM columns past the window rows) get (m = +inf, 1/l = 0): they add 0
            for (int r = et; r < rc; r += 128)
                sstat[g & 1][r] = r < R ? stats[(size_t)(b * G + g) * R + r] : make_float2(INFINITY, 0.0f);
            epi_bar();
            const float4* st4 = reinterpret_cast<const float4*>(sstat[g & 1]);
            for (int i = 0; i < nt; ++i) {
                const int it = g * nt + i, acc = it & 1;
                wait_or_trap(&tfull[acc], (it >> 1) & 1);
                umma::fence_after();
                float a4[4] = {0.0f, 0.0f, 0.0f, 0.0f};  // fixed order: (a0 + a1) + (a2 + a3) at the end
#pragma unroll 1
                for (int cc = 0; cc < rc / 32; ++cc) {
                    float v[32];
                    umma::ld32(tbase + ((uint32_t)(quarter * 32) << 16) + acc * rc + cc * 32, v);
#pragma unroll
                    for (int c = 0; c < 32; c += 2) {
                        const float4 ml = st4[(cc * 32 + c) >> 1];  // (m, 1/l) of rows c, c+1
                        a4[c & 3] += ex2(fmaf(v[c], scale_log2, -ml.x)) * ml.y;
                        a4[(c + 1) & 3] += ex2(fmaf(v[c + 1], scale_log2, -ml.z)) * ml.w;
                    }
                }
                const float a = (a4[0] + a4[1]) + (a4[2] + a4[3]);
                umma::fence_before();
                __syncwarp();
                if (lane == 0) umma::mbar_arrive(&tempty[acc]);
                salpha[i][row] = g == 0 ? a : salpha[i][row] + a;
            }
        }
        for (int i = 0; i < nt; ++i) {
            const int j = (t0 + i) * kKT + row;
            if (j < Lc) alpha[(size_t)b * Lc + j] = salpha[i][row];
        }
    }
    __syncthreads();
    if (warp == 1) {
        umma::fence_after();
        umma::tmem_free(tbase, ncols);
    }
}

// ---------------------------------------------------------------------------- top-k + buckets
// Multi-CTA top-m of ordered(alpha) per sequence (r02: the one-CTA-per-sequence version took 258 us
// per layer): 3 radix levels of 11 / 11 / 10 bits, each a histogram over all CTAs (shared-memory
// histogram, then global atomics) and one digit search per sequence; then per-CTA counts of the keys
// above / at the threshold, one scan per sequence, and the ordered keep writes.  Ties at the
// threshold key -> lowest index (A21): the first (m - #greater) equal keys in index order.
constexpr int kTkThreads = 256;
constexpr int kTkChunk = 2048;   // candidates per CTA
constexpr int kTkBins = 2048;

__device__ __forceinline__ int tk_shift(int level) { return level == 0 ? 21 : level == 1 ? 10 : 0; }
__device__ __forceinline__ uint32_t tk_bins(int level) { return level == 2 ? 1024u : 2048u; }

// tstate[b] = {prefix, need, -, -}; hist [B][kTkBins] zero on entry
__global__ void __launch_bounds__(kTkThreads) topk_hist_kernel(const float* __restrict__ alpha, int Lc, int level,
                                                              const uint32_t* __restrict__ tstate,
                                                              uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[kTkBins];
    const int b = blockIdx.y;
    const int shift = tk_shift(level);
    const uint32_t hmask = level == 0 ? 0u : (0xffffffffu << (tk_shift(level - 1)));
    const uint32_t prefix = tstate[b * 4];
    for (int i = threadIdx.x; i < kTkBins; i += kTkThreads) h[i] = 0u;
    __syncthreads();
    const float* a = alpha + (size_t)b * Lc;
    const int j0 = blockIdx.x * kTkChunk, j1 = min(Lc, j0 + kTkChunk);
    const uint32_t dmask = tk_bins(level) - 1u;
#pragma unroll 4
    for (int j = j0 + threadIdx.x; j < j1; j += kTkThreads) {
        const uint32_t k = ordered_key(a[j]);
        if ((k & hmask) == prefix) atomicAdd(&h[(k >> shift) & dmask], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < (int)tk_bins(level); i += kTkThreads)
        if (h[i]) atomicAdd(&hist[(size_t)b * kTkBins + i], h[i]);
}

// digit d with (count above d) < need <= (count above d) + hist[d]; prefix |= d << shift; zero hist
__global__ void __launch_bounds__(1024) topk_digit_kernel(int level, uint32_t* __restrict__ tstate,
                                                         uint32_t* __restrict__ hist) {
    __shared__ uint32_t ws32[32];
    __shared__ uint32_t s_d, s_need;
    const int b = blockIdx.x, tid = threadIdx.x;
    const uint32_t nb = tk_bins(level);
    uint32_t* hb = hist + (size_t)b * kTkBins;
    // thread t owns the 2 bins nb-1-2t, nb-2-2t (descending digits in thread order)
    uint32_t c[2], sum = 0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int bin = (int)nb - 1 - (2 * tid + k);
        c[k] = bin >= 0 ? hb[bin] : 0u;
        sum += c[k];
    }
    uint32_t tot;
    uint32_t above = block_incl_sum<uint32_t>(sum, ws32, &tot) - sum;
    const uint32_t need = tstate[b * 4 + 1];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int bin = (int)nb - 1 - (2 * tid + k);
        if (bin >= 0 && above < need && above + c[k] >= need) {
            s_d = (uint32_t)bin;
            s_need = need - above;
        }
        above += c[k];
    }
    __syncthreads();
    for (int i = tid; i < kTkBins; i += 1024) hb[i] = 0u;
    if (tid == 0) {
        tstate[b * 4] |= s_d << tk_shift(level);
        tstate[b * 4 + 1] = s_need;
    }
}

// per CTA: keys above / equal to the threshold T = tstate[b].prefix
__global__ void __launch_bounds__(kTkThreads) topk_count_kernel(const float* __restrict__ alpha, int Lc,
                                                               const uint32_t* __restrict__ tstate,
                                                               uint32_t* __restrict__ cnt) {
    __shared__ uint32_t ws32[32];
    const int b = blockIdx.y;
    const uint32_t T = tstate[b * 4];
    const float* a = alpha + (size_t)b * Lc;
    const int j0 = blockIdx.x * kTkChunk, j1 = min(Lc, j0 + kTkChunk);
    uint32_t v = 0;
#pragma unroll 4
    for (int j = j0 + threadIdx.x; j < j1; j += kTkThreads) {
        const uint32_t k = ordered_key(a[j]);
        v += k > T ? (1u << 16) : (k == T ? 1u : 0u);  // (gt << 16) | eq, both <= kTkChunk
    }
    uint32_t tot;
    block_incl_sum<uint32_t>(v, ws32, &tot);
    if (threadIdx.x == 0) cnt[(size_t)b * gridDim.x + blockIdx.x] = tot;
}

// ordered keep writes: the CTA's first output slot and equal-key rank from the counts of the CTAs before
__global__ void __launch_bounds__(kTkThreads) topk_write_kernel(const float* __restrict__ alpha, int Lc, int m,
                                                               const uint32_t* __restrict__ tstate,
                                                               const uint32_t* __restrict__ cnt,
                                                               int32_t* __restrict__ keep) {
    __shared__ uint32_t ws32[32];
    __shared__ uint32_t s_gt, s_eq;
    const int b = blockIdx.y, tid = threadIdx.x;
    const uint32_t T = tstate[b * 4], need = tstate[b * 4 + 1];
    if (tid < 32) {  // counts of the CTAs before this one
        uint32_t g = 0, e = 0;
        for (int x = tid; x < (int)blockIdx.x; x += 32) {
            const uint32_t c = cnt[(size_t)b * gridDim.x + x];
            g += c >> 16;
            e += c & 0xffffu;
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            g += __shfl_xor_sync(0xffffffffu, g, o);
            e += __shfl_xor_sync(0xffffffffu, e, o);
        }
        if (tid == 0) {
            s_gt = g;
            s_eq = e;
        }
    }
    __syncthreads();
    const float* a = alpha + (size_t)b * Lc;
    int32_t* kp = keep + (size_t)b * m;
    // thread t owns the contiguous elements [j0 + 8t, j0 + 8t + 8)
    const int j0 = blockIdx.x * kTkChunk + tid * (kTkChunk / kTkThreads);
    uint32_t k8[kTkChunk / kTkThreads];
    uint32_t eq = 0;
#pragma unroll
    for (int u = 0; u < kTkChunk / kTkThreads; ++u) {
        const int j = j0 + u;
        k8[u] = j < Lc ? ordered_key(a[j]) : 0u;
        eq += (j < Lc && k8[u] == T) ? 1u : 0u;
    }
    uint32_t tot;
    uint32_t e = s_eq + block_incl_sum<uint32_t>(eq, ws32, &tot) - eq;  // equal keys before this thread's
    uint32_t mine = 0;
    {
        uint32_t ee = e;
#pragma unroll
        for (int u = 0; u < kTkChunk / kTkThreads; ++u) {
            const int j = j0 + u;
            if (j < Lc && (k8[u] > T || (k8[u] == T && ee++ < need))) ++mine;
        }
    }
    // kept before this CTA = its gt count + min(its equal count, need)
    uint32_t pos = s_gt + min(s_eq, need) + block_incl_sum<uint32_t>(mine, ws32, &tot) - mine;
#pragma unroll
    for (int u = 0; u < kTkChunk / kTkThreads; ++u) {
        const int j = j0 + u;
        if (j < Lc && (k8[u] > T || (k8[u] == T && e++ < need))) kp[pos++] = j;
    }
}


// One CTA per sequence.  Keys: ordered(alpha) (NaN ranks last, reading A14's rule); the m-th largest
// key T by a 4-pass 8-bit radix select; kept = key > T, or key == T among the first (m - #greater)
// in index order (ties -> lowest index, A21).  Then the retained buckets: kept token i lies in
// sentence s_i; a bucket starts wherever s_i changes (sentences without a kept token vanish, A25).
// Every pass reads alpha coalesced: warp w owns the contiguous range [w*C, (w+1)*C), lane = element.
constexpr int kTopThreads = 1024;
constexpr int kTopWarps = kTopThreads / 32;

__global__ void __launch_bounds__(kTopThreads) retain_buckets_kernel(int m, const int32_t* __restrict__ off,
                                                                     int off_stride, const int32_t* __restrict__ S,
                                                                     const int32_t* __restrict__ keep,
                                                                     int32_t* __restrict__ roff,
                                                                     int32_t* __restrict__ rsid,
                                                                     int32_t* __restrict__ rS, int off_cap) {
    __shared__ uint32_t wgt[kTopWarps];
    __shared__ int32_t s_last[kTopWarps];
    const int b = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int32_t* kp = keep + (size_t)b * m;
    // buckets: sentence of every kept token (binary search in the prompt offsets), starts where it changes
    const int Sb = S[b];
    const int32_t* o = off + (size_t)b * off_stride;
    extern __shared__ int32_t soff[];  // the prompt's offsets, when they fit (dynamic smem sized by the launcher)
    if (Sb + 1 <= off_cap) {
        for (int i = tid; i <= Sb; i += kTopThreads) soff[i] = o[i];
        __syncthreads();
        o = soff;
    }
    const int Cm = (m + kTopWarps - 1) / kTopWarps;
    const int i0 = min(m, warp * Cm), i1 = min(m, i0 + Cm);
    auto sent_of = [&](int t) {  // largest s with o[s] <= t
        int lo = 0, hi = Sb - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (o[mid] <= t) lo = mid; else hi = mid - 1;
        }
        return lo;
    };
    uint32_t nstart = 0;
    int32_t last = -1;
    for (int x0 = i0; x0 < i1; x0 += 32) {
        const int x = x0 + lane;
        const int s = x < i1 ? sent_of(kp[x]) : -1;
        int prev = __shfl_up_sync(0xffffffffu, s, 1);
        if (lane == 0) prev = last;
        nstart += __popc(__ballot_sync(0xffffffffu, x < i1 && s != prev));
        last = __shfl_sync(0xffffffffu, s, 31);
        const int nv = min(32, i1 - x0);
        last = __shfl_sync(0xffffffffu, s, nv - 1);
    }
    if (lane == 0) {
        wgt[warp] = nstart;
        s_last[warp] = last;
    }
    __syncthreads();
    // a warp's first token starts a bucket unless the previous non-empty warp ended in the same sentence
    uint32_t sp = 0;
    int32_t carry = -1;
    for (int w = 0; w < warp; ++w) {
        if (s_last[w] >= 0) carry = s_last[w];
    }
    for (int w = 0; w < warp; ++w) sp += wgt[w];
    // (the per-warp counts above treated each warp's first token as a start; subtract the duplicates)
    __shared__ uint32_t s_dup[kTopWarps];
    if (lane == 0) {
        int32_t first = i0 < i1 ? sent_of(kp[i0]) : -2;
        s_dup[warp] = (i0 < i1 && first == carry) ? 1u : 0u;
    }
    __syncthreads();
    for (int w = 0; w <= warp; ++w) sp -= (w < warp) ? s_dup[w] : 0u;
    int32_t* ro = roff + (size_t)b * (m + 1);
    int32_t* rs = rsid + (size_t)b * m;
    last = s_dup[warp] ? carry : -1;
    for (int x0 = i0; x0 < i1; x0 += 32) {
        const int x = x0 + lane;
        const int s = x < i1 ? sent_of(kp[x]) : -1;
        int prev = __shfl_up_sync(0xffffffffu, s, 1);
        if (lane == 0) prev = last;
        const bool start = x < i1 && s != prev;
        const unsigned sm_ = __ballot_sync(0xffffffffu, start);
        if (start) {
            const uint32_t q = sp + __popc(sm_ & ((1u << lane) - 1u));
            ro[q] = x;
            rs[q] = s;
        }
        sp += __popc(sm_);
        const int nv = min(32, i1 - x0);
        last = __shfl_sync(0xffffffffu, s, nv - 1);
    }
    __syncthreads();
    if (tid == kTopThreads - 1) {
        uint32_t tot = 0;
        for (int w = 0; w < kTopWarps; ++w) tot += wgt[w] - s_dup[w];
        ro[tot] = m;
        rS[b] = (int32_t)tot;
    }
}

// pool[b][g][i] = X[b][g][keep[b][i]] for K and V (16 bytes per thread)
__global__ void retain_gather_kernel(const __nv_bfloat16* __restrict__ K, const __nv_bfloat16* __restrict__ V, int G,
                                     int L, int d, int m, const int32_t* __restrict__ keep, __nv_bfloat16* __restrict__ PK,
                                     __nv_bfloat16* __restrict__ PV) {
    const int g = blockIdx.y, b = blockIdx.z;
    const int per_row = d / 8;
    const size_t n = (size_t)m * per_row;
    const int32_t* kp = keep + (size_t)b * m;
    const uint4* k4 = reinterpret_cast<const uint4*>(K + (size_t)(b * G + g) * L * d);
    const uint4* v4 = reinterpret_cast<const uint4*>(V + (size_t)(b * G + g) * L * d);
    uint4* pk = reinterpret_cast<uint4*>(PK + (size_t)(b * G + g) * m * d);
    uint4* pv = reinterpret_cast<uint4*>(PV + (size_t)(b * G + g) * m * d);
    for (size_t x = (size_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (size_t)gridDim.x * blockDim.x) {
        const size_t i = x / per_row, c = x % per_row;
        const size_t src = (size_t)kp[i] * per_row + c;
        pk[x] = k4[src];
        pv[x] = v4[src];
    }
}

// ---------------------------------------------------------------------------- host side
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encoder() {
    static EncodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiled>(p);
    });
    return fn;
}

// bf16 tensor [outer...][inner], inner extent `d`, box {64, rows...}, 128-byte swizzle
bool make_map(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides_bytes,
              const cuuint32_t* box) {
    EncodeTiled enc = encoder();
    if (!enc) return false;
    cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims, strides_bytes, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

size_t retain_scratch_floats(int B, int G, int L, int N, int grp) {
    const int R = N * grp, nrb = (R + 127) / 128;
    const int nchunk = (L + kKT - 1) / kKT;  // upper bound (chunk_tiles >= 1)
    const size_t topk = 4 * (size_t)B + (size_t)B * kTkBins + (size_t)B * ((L + kTkChunk - 1) / kTkChunk);
    return (size_t)B * G * nrb * nchunk * 128 * 2 + (size_t)B * G * R * 2 + topk;
}

bool retain_supported(int d, int N, int grp) {
    const int R = N * grp;
    return (d == 64 || d == 128) && N >= 1 && R % 16 == 0 && R <= 256 && N <= 256;
}

cudaError_t launch_retain(const RetainArgs& a, cudaStream_t st) {
    const int R = a.N * a.grp, nrb = (R + 127) / 128, DH = a.d / 64, Lc = a.L - a.N;
    const int Hq = a.G * a.grp;
    const float scale_log2 = (float)(1.0 / sqrt((double)a.d) * 1.4426950408889634);
    // tensor maps: K [B*G*L][d]; window queries [B*N][Hq][d] (box rows = (w, head in group))
    CUtensorMap tmK, tmQa, tmQb;
    {
        cuuint64_t dims[2] = {(cuuint64_t)a.d, (cuuint64_t)a.B * a.G * a.L};
        cuuint64_t strides[1] = {(cuuint64_t)a.d * 2};
        cuuint32_t box[2] = {64, (cuuint32_t)kKT};
        if (!make_map(&tmK, a.K, 2, dims, strides, box)) return cudaErrorInvalidValue;
    }
    const int wbox = std::min(a.N, 128 / a.grp);
    {
        cuuint64_t dims[3] = {(cuuint64_t)a.d, (cuuint64_t)Hq, (cuuint64_t)a.B * a.N};
        cuuint64_t strides[2] = {(cuuint64_t)a.d * 2, (cuuint64_t)Hq * a.d * 2};
        cuuint32_t boxa[3] = {64, (cuuint32_t)a.grp, (cuuint32_t)wbox};
        cuuint32_t boxb[3] = {64, (cuuint32_t)a.grp, (cuuint32_t)a.N};
        if (!make_map(&tmQa, a.q_window, 3, dims, strides, boxa)) return cudaErrorInvalidValue;
        if (!make_map(&tmQb, a.q_window, 3, dims, strides, boxb)) return cudaErrorInvalidValue;
    }
    // pass A: chunks of keys per (b, g, row block), sized to fill the SMs about twice
    const int ntiles = (a.L + kKT - 1) / kKT;
    const int units = a.B * a.G * nrb;
    const int want = std::max(1, 2 * kNumSMs / std::max(1, units));
    const int chunk_tiles = std::max(1, (ntiles + want - 1) / want);
    const int nchunk = (ntiles + chunk_tiles - 1) / chunk_tiles;
    float2* part = reinterpret_cast<float2*>(a.scratch);
    float2* stats = part + (size_t)a.B * a.G * nrb * nchunk * 128;
    const size_t smemA = 1024 + (size_t)DH * kHalf * (1 + kStages);
    const int qhalf = (R * 128 + 1023) / 1024 * 1024;
    const size_t smemB = 1024 + (size_t)DH * qhalf + (size_t)DH * kHalf * kStages;
    cudaError_t e;
    if (DH == 2) {
        if ((e = ensure_smem((const void*)alpha_rowstats_kernel<2>, smemA)) != cudaSuccess) return e;
        alpha_rowstats_kernel<2><<<dim3(nchunk, a.G * nrb, a.B), kThreads, smemA, st>>>(
            tmQa, tmK, a.L, a.N, a.grp, a.G, R, nrb, wbox, chunk_tiles, scale_log2, part);
    } else {
        if ((e = ensure_smem((const void*)alpha_rowstats_kernel<1>, smemA)) != cudaSuccess) return e;
        alpha_rowstats_kernel<1><<<dim3(nchunk, a.G * nrb, a.B), kThreads, smemA, st>>>(
            tmQa, tmK, a.L, a.N, a.grp, a.G, R, nrb, wbox, chunk_tiles, scale_log2, part);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    alpha_rowcombine_kernel<<<dim3(a.G, a.B), 256, 0, st>>>(part, a.G, R, nrb, nchunk, stats);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // pass B: every SM one CTA, each a run of key tiles of one sequence, all KV heads
    const int ntc = (Lc + kKT - 1) / kKT;
    const int per_b = std::max(1, 2 * kNumSMs / a.B);  // two CTAs per SM
    const int tiles_per_cta = std::min(kMaxTiles, std::max(1, (ntc + per_b - 1) / per_b));
    const int nctb = (ntc + tiles_per_cta - 1) / tiles_per_cta;
    if (DH == 2) {
        if ((e = ensure_smem((const void*)alpha_colsum_kernel<2>, smemB)) != cudaSuccess) return e;
        alpha_colsum_kernel<2><<<dim3(nctb, a.B), kThreads, smemB, st>>>(tmQb, tmK, a.L, a.N, a.grp, a.G, R, Lc,
                                                                          tiles_per_cta, qhalf, scale_log2, stats, a.alpha);
    } else {
        if ((e = ensure_smem((const void*)alpha_colsum_kernel<1>, smemB)) != cudaSuccess) return e;
        alpha_colsum_kernel<1><<<dim3(nctb, a.B), kThreads, smemB, st>>>(tmQb, tmK, a.L, a.N, a.grp, a.G, R, Lc,
                                                                          tiles_per_cta, qhalf, scale_log2, stats, a.alpha);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // top-m: 3 radix levels over all CTAs, then counts, then the ordered keep writes
    {
        const int nblk = (Lc + kTkChunk - 1) / kTkChunk;
        uint32_t* ts = reinterpret_cast<uint32_t*>(stats + (size_t)a.B * a.G * R);  // [B][4]
        uint32_t* th = ts + 4 * a.B;                                                // [B][kTkBins]
        uint32_t* tc = th + (size_t)a.B * kTkBins;                                  // [B][nblk]
        std::vector<uint32_t> init(4 * a.B, 0u);
        for (int b = 0; b < a.B; ++b) init[4 * b + 1] = (uint32_t)a.m;
        if ((e = cudaMemcpyAsync(ts, init.data(), sizeof(uint32_t) * 4 * a.B, cudaMemcpyHostToDevice, st)) != cudaSuccess)
            return e;
        if ((e = cudaMemsetAsync(th, 0, sizeof(uint32_t) * a.B * kTkBins, st)) != cudaSuccess) return e;
        for (int level = 0; level < 3; ++level) {
            topk_hist_kernel<<<dim3(nblk, a.B), kTkThreads, 0, st>>>(a.alpha, Lc, level, ts, th);
            topk_digit_kernel<<<a.B, 1024, 0, st>>>(level, ts, th);
        }
        topk_count_kernel<<<dim3(nblk, a.B), kTkThreads, 0, st>>>(a.alpha, Lc, ts, tc);
        topk_write_kernel<<<dim3(nblk, a.B), kTkThreads, 0, st>>>(a.alpha, Lc, a.m, ts, tc, a.keep);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    // buckets (the prompt's sentence offsets in shared memory when they fit in 96 KB)
    const int off_cap = std::min(a.off_stride, 96 * 1024 / 4);
    if ((e = ensure_smem((const void*)retain_buckets_kernel, (size_t)off_cap * 4)) != cudaSuccess) return e;
    retain_buckets_kernel<<<a.B, kTopThreads, (size_t)off_cap * 4, st>>>(a.m, a.off, a.off_stride, a.S, a.keep, a.roff,
                                                                        a.rsid, a.rS, off_cap);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    const int blocks = std::max(1, std::min(64, (a.m * a.d / 8 + 255) / 256));
    retain_gather_kernel<<<dim3(blocks, a.G, a.B), 256, 0, st>>>(a.K, a.V, a.G, a.L, a.d, a.m, a.keep, a.PK, a.PV);
    return cudaGetLastError();
}

}  // namespace skv
