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
// One thread-block cluster of kCL CTAs per (b, g) unit.  The unit's gathered token range
// [0, ntok) is cut into 64-token chunks; CTA r of the cluster takes a contiguous run of chunks
// and streams them through a 2-stage shared-memory pipeline (bulk copies of chunk i+1 in flight
// while chunk i is computed), keeping an online softmax (running max / sum in the log2 domain)
// for all grp query heads of the KV head (GQA: every K/V byte is read once for grp heads).
// The kCL partial results are merged through distributed shared memory -- no workspace in HBM,
// no second launch.
#include "device_util.cuh"
#include "skv_internal.cuh"

namespace skv {
SKV_TRACE_DEFINE(attend)
}  // namespace skv

#include "attend_core.cuh"

namespace skv {

int attend_chunk_tokens(int) { return kAttC; }

template <int D, int GRP>
__global__ void __cluster_dims__(kCL, 1, 1) __launch_bounds__(kAttThreads, GRP <= 4 ? 2 : 1)
attend_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ K,
              const __nv_bfloat16* __restrict__ V, int G, int L, const int32_t* __restrict__ sel_src,
              const int32_t* __restrict__ sel_tokoff, const int32_t* __restrict__ sel_count, int tau,
              float* __restrict__ out, float scale_log2) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    AttSmem<D, GRP>& sm = *reinterpret_cast<AttSmem<D, GRP>*>(smem_raw);
    cg::cluster_group cluster = cg::this_cluster();

    const int rank = (int)cluster.block_rank();
    const int g = blockIdx.y, b = blockIdx.z;
    const int unit = b * G + g;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int Hq = G * GRP;
    SKV_TRACE_POINT(0);
    if (tid == 0)
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&sm.bar[s], 1);
            sm.done[s] = 0u;
        }
    if (tid < kAttWarps * GRP) {
        (&sm.mw[0][0])[tid] = -INFINITY;
        (&sm.lw[0][0])[tid] = 0.0f;
    }
    pdl_wait();
    const int count = sel_count[unit];
    const __nv_bfloat16* Kh = K + (size_t)unit * L * D;
    const __nv_bfloat16* Vh = V + (size_t)unit * L * D;
    // selection metadata -> shared memory (parallel loads; the gather then never touches L2)
    int32_t* tok = reinterpret_cast<int32_t*>(smem_raw + sizeof(AttSmem<D, GRP>));  // [count + 1]
    int32_t* srcs = tok + (tau + 1);                                                // [count]
    {
        const int32_t* gt = sel_tokoff + (size_t)unit * (tau + 1);
        const int32_t* gs = sel_src + (size_t)unit * tau;
        for (int i = tid; i <= count; i += kAttThreads) {
            tok[i] = gt[i];
            if (i < count) srcs[i] = gs[i];
        }
    }
    __syncthreads();
    SKV_TRACE_POINT(1);
    attend_body<D, GRP>(sm, tok, srcs, count, Kh, Vh, q, out, b, g, G, scale_log2, cluster);
}

template <int D, int GRP>
static cudaError_t launch_one(dim3 grid, cudaStream_t st, const __nv_bfloat16* q, const __nv_bfloat16* K,
                              const __nv_bfloat16* V, int G, int L, const int32_t* sel_src,
                              const int32_t* sel_tokoff, const int32_t* sel_count, int tau, float* out,
                              float scale_log2) {
    const size_t smem = sizeof(AttSmem<D, GRP>) + sizeof(int32_t) * (2 * (size_t)tau + 1);
    static size_t configured = 0;
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(attend_kernel<D, GRP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(attend_kernel<D, GRP>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    return launch_pdl(attend_kernel<D, GRP>, grid, dim3(kAttThreads), smem, st, q, K, V, G, L, sel_src, sel_tokoff,
                      sel_count, tau, out, scale_log2);
}

cudaError_t launch_attend(const __nv_bfloat16* q, const __nv_bfloat16* K, const __nv_bfloat16* V, int B, int G,
                          int grp, int d, int L, const int32_t* sel_src, const int32_t* sel_tokoff,
                          const int32_t* sel_count, int tau, float* out, cudaStream_t st) {
    dim3 grid(kCL, G, B);
    const float scale_log2 = (float)(1.0 / sqrt((double)d) * 1.4426950408889634);
#define SKV_ATT(DV, GV) \
    return launch_one<DV, GV>(grid, st, q, K, V, G, L, sel_src, sel_tokoff, sel_count, tau, out, scale_log2)
    if (d == 128) {
        switch (grp) {
            case 1: SKV_ATT(128, 1);
            case 2: SKV_ATT(128, 2);
            case 4: SKV_ATT(128, 4);
            case 8: SKV_ATT(128, 8);
        }
    } else {
        switch (grp) {
            case 1: SKV_ATT(64, 1);
            case 2: SKV_ATT(64, 2);
            case 4: SKV_ATT(64, 4);
            case 8: SKV_ATT(64, 8);
        }
    }
#undef SKV_ATT
    return cudaErrorInvalidValue;
}

}  // namespace skv
