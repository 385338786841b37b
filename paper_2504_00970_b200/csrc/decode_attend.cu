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
attend_kernel(const __nv_bfloat16* __restrict__ q, KvSrc kv, int G, SelBufs sel, QsState qs,
              float* __restrict__ out, float scale_log2) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    AttSmem<D, GRP>& sm = *reinterpret_cast<AttSmem<D, GRP>*>(smem_raw);
    cg::cluster_group cluster = cg::this_cluster();

    const int g = blockIdx.y, b = blockIdx.z;
    const int unit = b * G + g;
    const int tid = threadIdx.x;
    const int tau = sel.tau;
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
    if (cluster.block_rank() == 0) qs_update_unit(q, qs.input_token, qs.bset, qs.nb, qs.Sq, qs.cnt, b, g, G, GRP, D, tid, kAttThreads);
    const int cur = sel.parity[unit] ^ 1;  // the selection made by this step's decode_select
    const int count = *sel.count_of(cur, unit);
    const size_t base = (size_t)unit * kv.unit_stride + (size_t)cur * kv.slot_stride;
    const __nv_bfloat16* Kh = kv.K + base * D;
    const __nv_bfloat16* Vh = kv.V + base * D;
    // selection metadata -> shared memory (parallel loads; the gather then never touches L2)
    int32_t* tok = reinterpret_cast<int32_t*>(smem_raw + sizeof(AttSmem<D, GRP>));  // [count + 1]
    int32_t* srcs = tok + (tau + 1);                                                // [count]
    {
        const int32_t* gt = sel.tok_of(cur, unit);
        const int32_t* gs = sel.src_of(cur, unit);
        for (int i = tid; i <= count; i += kAttThreads) {
            tok[i] = gt[i];
            if (i < count) srcs[i] = gs[i];
        }
    }
    __syncthreads();
    SKV_TRACE_POINT(1);
    attend_body<D, GRP>(sm, tok, srcs, count, Kh, Vh, q, out, b, g, G, scale_log2, cluster);
    // every CTA of the cluster has read the parity (attend_body ends with a cluster barrier)
    if (cluster.block_rank() == 0 && tid == 0) sel.parity[unit] = cur;
}

// Host residency (D3 + D4): K/V live in the mapped pinned host store (P3); each selected sentence is
// resolved against the previous step's selection of the unit (binary search of its id): a hit is
// re-read from the previous HBM working-set slot, a miss from the host over PCIe; the staged chunks
// are written through to the current slot (attend_core.cuh, HostWs).
template <int D, int GRP>
__global__ void __cluster_dims__(kCL, 1, 1) __launch_bounds__(kAttThreads, GRP <= 4 ? 2 : 1)
attend_host_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* Khost, const __nv_bfloat16* Vhost,
                   int L, __nv_bfloat16* wsK, __nv_bfloat16* wsV, int G, SelBufs sel,
                   unsigned long long* __restrict__ ledger, QsState qs, float* __restrict__ out, float scale_log2) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    AttSmem<D, GRP>& sm = *reinterpret_cast<AttSmem<D, GRP>*>(smem_raw);
    cg::cluster_group cluster = cg::this_cluster();
    const int g = blockIdx.y, b = blockIdx.z;
    const int unit = b * G + g;
    const int tid = threadIdx.x;
    const int tau = sel.tau;
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
    if (cluster.block_rank() == 0) qs_update_unit(q, qs.input_token, qs.bset, qs.nb, qs.Sq, qs.cnt, b, g, G, GRP, D, tid, kAttThreads);
    const int prev = sel.parity[unit], cur = prev ^ 1;
    const int count = *sel.count_of(cur, unit);
    const int pcount = *sel.count_of(prev, unit);
    int32_t* tok = reinterpret_cast<int32_t*>(smem_raw + sizeof(AttSmem<D, GRP>));  // [tau + 1]
    int32_t* srcs = tok + (tau + 1);                                                // [tau]
    int32_t* pids = srcs + tau;                                                     // [tau]
    int32_t* ptok = pids + tau;                                                     // [tau + 1]
    {
        const int32_t* gt = sel.tok_of(cur, unit);
        const int32_t* pi = sel.ids_of(prev, unit);
        const int32_t* pt = sel.tok_of(prev, unit);
        for (int i = tid; i <= max(count, pcount); i += kAttThreads) {
            if (i <= count) tok[i] = gt[i];
            if (i < pcount) pids[i] = pi[i];
            if (i <= pcount) ptok[i] = pt[i];
        }
    }
    __syncthreads();
    {
        const int32_t* gi = sel.ids_of(cur, unit);
        const int32_t* gs = sel.src_of(cur, unit);
        for (int i = tid; i < count; i += kAttThreads) {
            const int id = gi[i];
            int lo = 0, hi = pcount;  // first index with pids >= id
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (pids[mid] < id) lo = mid + 1; else hi = mid;
            }
            srcs[i] = (lo < pcount && pids[lo] == id) ? -(ptok[lo] + 1) : gs[i];
        }
    }
    __syncthreads();
    HostWs ws;
    ws.prevK = wsK + ((size_t)unit * 2 + prev) * tau * D;
    ws.prevV = wsV + ((size_t)unit * 2 + prev) * tau * D;
    ws.curK = wsK + ((size_t)unit * 2 + cur) * tau * D;
    ws.curV = wsV + ((size_t)unit * 2 + cur) * tau * D;
    ws.ledger = ledger;
    const __nv_bfloat16* Kh = Khost + (size_t)unit * L * D;
    const __nv_bfloat16* Vh = Vhost + (size_t)unit * L * D;
    attend_body<D, GRP, true>(sm, tok, srcs, count, Kh, Vh, q, out, b, g, G, scale_log2, cluster, ws);
    if (cluster.block_rank() == 0 && tid == 0) sel.parity[unit] = cur;
}

template <int D, int GRP>
static cudaError_t launch_host_one(dim3 grid, cudaStream_t st, const __nv_bfloat16* q, const __nv_bfloat16* Kh,
                                   const __nv_bfloat16* Vh, int L, __nv_bfloat16* wsK, __nv_bfloat16* wsV, int G,
                                   SelBufs sel, unsigned long long* ledger, QsState qs, float* out, float scale_log2) {
    const size_t smem = sizeof(AttSmem<D, GRP>) + sizeof(int32_t) * (4 * (size_t)sel.tau + 2);
    static size_t configured = 0;
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(attend_host_kernel<D, GRP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(attend_host_kernel<D, GRP>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    return launch_pdl(attend_host_kernel<D, GRP>, grid, dim3(kAttThreads), smem, st, q, Kh, Vh, L, wsK, wsV, G, sel,
                      ledger, qs, out, scale_log2);
}

cudaError_t launch_attend_host(const __nv_bfloat16* q, const __nv_bfloat16* Kh, const __nv_bfloat16* Vh, int L,
                               __nv_bfloat16* wsK, __nv_bfloat16* wsV, int B, int G, int grp, int d, SelBufs sel,
                               unsigned long long* ledger, QsState qs, float* out, cudaStream_t st) {
    dim3 grid(kCL, G, B);
    const float scale_log2 = (float)(1.0 / sqrt((double)d) * 1.4426950408889634);
#define SKV_ATH(DV, GV) return launch_host_one<DV, GV>(grid, st, q, Kh, Vh, L, wsK, wsV, G, sel, ledger, qs, out, scale_log2)
    if (d == 128) {
        switch (grp) {
            case 1: SKV_ATH(128, 1);
            case 2: SKV_ATH(128, 2);
            case 4: SKV_ATH(128, 4);
            case 8: SKV_ATH(128, 8);
        }
    } else {
        switch (grp) {
            case 1: SKV_ATH(64, 1);
            case 2: SKV_ATH(64, 2);
            case 4: SKV_ATH(64, 4);
            case 8: SKV_ATH(64, 8);
        }
    }
#undef SKV_ATH
    return cudaErrorInvalidValue;
}

template <int D, int GRP>
static cudaError_t launch_one(dim3 grid, cudaStream_t st, const __nv_bfloat16* q, KvSrc kv, int G, SelBufs sel,
                              QsState qs, float* out, float scale_log2) {
    const size_t smem = sizeof(AttSmem<D, GRP>) + sizeof(int32_t) * (2 * (size_t)sel.tau + 1);
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
    return launch_pdl(attend_kernel<D, GRP>, grid, dim3(kAttThreads), smem, st, q, kv, G, sel, qs, out, scale_log2);
}

cudaError_t launch_attend(const __nv_bfloat16* q, KvSrc kv, int B, int G, int grp, int d, SelBufs sel, QsState qs,
                          float* out, cudaStream_t st) {
    dim3 grid(kCL, G, B);
    const float scale_log2 = (float)(1.0 / sqrt((double)d) * 1.4426950408889634);
#define SKV_ATT(DV, GV) return launch_one<DV, GV>(grid, st, q, kv, G, sel, qs, out, scale_log2)
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
