// skv_internal.cuh -- shared declarations of the SentenceKV sm_100a kernels and the runtime
// context behind the C ABI (include/sentencekv.h).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/sentencekv.h"

namespace skv {

constexpr int kMaxBoundary = 64;

// Double-buffered selection of one layer.  Slot `parity[unit]` holds the previous step's
// selection; decode_select writes slot parity^1; decode_attend flips parity at its end.  (The
// previous selection is what the host-residency gather reuses and what the fused kernel
// prefetches.)  The flip happens on the device, so replaying a captured step stays consistent.
struct SelBufs {
    int32_t* ids;     // [2][units][tau]    ascending selected sentence ids
    int32_t* tokoff;  // [2][units][tau+1]  prefix sums of the selected lengths (gathered offsets)
    int32_t* src;     // [2][units][tau]    first K/V row of each selected sentence in the attended store
    int32_t* count;   // [2][units]         selected sentences
    int32_t* parity;  // [units]
    int units, tau;
    __host__ __device__ int32_t* ids_of(int slot, int u) const { return ids + ((size_t)slot * units + u) * tau; }
    __host__ __device__ int32_t* tok_of(int slot, int u) const { return tokoff + ((size_t)slot * units + u) * (tau + 1); }
    __host__ __device__ int32_t* src_of(int slot, int u) const { return src + ((size_t)slot * units + u) * tau; }
    __host__ __device__ int32_t* count_of(int slot, int u) const { return count + (size_t)slot * units + u; }
};

// The deferred Eq. 2 state update of a layer (Sq += q_t or reset), done by the attend kernels
// after the step's scoring and selection (qs_update_unit in device_util.cuh).
struct QsState {
    const int32_t* input_token;  // [B]
    const int32_t* bset;
    int nb;
    float* Sq;                   // [B][Hq][d]
    int32_t* cnt;                // [B][G]
};

// Where decode_attend reads K/V rows: unit u, slot s, row r -> base + ((u * unit_stride) +
// s * slot_stride + r) * d.  Device residency: the caller's K/V (unit_stride = L, slot_stride = 0,
// rows = context tokens).  Host residency: the HBM working set (unit_stride = 2*tau,
// slot_stride = tau, rows = gathered positions).
struct KvSrc {
    const __nv_bfloat16* K;
    const __nv_bfloat16* V;
    long long unit_stride, slot_stride;
};
constexpr int kNumSMs = 148;

// Per-layer device state.  Sizes use the ctx shard: B = batch_count, G = kv_head_count,
// Hq = G * grp, Smax = sentence capacity of the current prompt.
struct LayerState {
    bool prefilled = false;
    bool selected = false;             // a decode_select ran since the prefill
    const int32_t* input_token = nullptr;  // of the last decode_select (its Eq. 2 update runs in attend)
    const __nv_bfloat16* K = nullptr;  // device residency: borrowed [B][G][L][d]
    const __nv_bfloat16* V = nullptr;
    __nv_bfloat16* E = nullptr;        // [B][G][Smax][d]  sentence embeddings (Eq. 1)
    float* Sq = nullptr;               // [B][Hq][d]       running query sum of Q_s (Eq. 2)
    int32_t* cnt = nullptr;            // [B][G]           |Q_s| (one copy per KV-head unit)
    float* scores = nullptr;           // [B][G][Smax]     last step's similarity scores
    SelBufs sel{};                     // double-buffered selection (see SelBufs)
    // host residency (P3 + D3)
    __nv_bfloat16* Kh = nullptr;       // pinned, mapped host [B][G][L][d] (full K/V)
    __nv_bfloat16* Vh = nullptr;
    size_t host_bytes = 0;             // bytes of each of Kh, Vh
    __nv_bfloat16* wsK = nullptr;      // HBM working set [B][G][2][tau][d] (gathered rows, 2 slots)
    __nv_bfloat16* wsV = nullptr;
    unsigned long long* ledger = nullptr;  // device: host->HBM bytes fetched by the gathers (cumulative)
    cudaEvent_t offload_done = nullptr;    // D2H copies of this layer completed
    bool host_ready = false;
    // persistent per-layer kernel: work queue + dependency counters + merge workspace
    uint32_t* lk_counters = nullptr;   // [3 + 3 * units]: ticket, exit_count, pad, score/select/attend done
    float* lk_part_ml = nullptr;       // [units][n_att][8][2]
    float* lk_part_o = nullptr;        // [units][n_att][8][d]
    int4* lk_cand = nullptr;           // [units][n_score_max][NL] local selection candidates
    int32_t* lk_cand_count = nullptr;  // [units][n_score_max]
    uint2* unit_hint = nullptr;        // [units] one-launch step kernel: band of the selection's crossing point
    int32_t* pc_pt = nullptr;          // host residency, one-launch kernel: page table [units][pages]
    int32_t* pc_own = nullptr;         // [units][slots]
    int32_t* pc_hand = nullptr;        // [units]
    int pc_pages = 0;
    int last_path = 0;                 // host residency: 1 = one-launch kernel (page cache), 2 = split kernels
};

}  // namespace skv

struct skv_ctx {
    skv_config cfg{};
    int B = 0, G = 0, Hq = 0, grp = 0, d = 0, tau = 0;
    std::string err;
    skv_status sticky = SKV_OK;
    int64_t launches = 0;

    // prompt state
    int L = 0;
    int Smax = 0;                      // sentence capacity per (b)
    int off_stride = 0;                // row stride of `off` (= L + 1)
    std::vector<int32_t> S_host;       // [B]
    int32_t* off = nullptr;            // device [B][L+1]
    int32_t* S_dev = nullptr;          // device [B]
    int32_t* bset = nullptr;           // device [kMaxBoundary]
    int n_bset = 0;

    std::vector<skv::LayerState> layer;
    int2* lk_items = nullptr;          // device work queue of the per-layer kernel (per prompt)
    int lk_n_items = 0;
    int lk_n_score_max = 0;            // SCORE items of the longest sequence (per-layer candidate lists)
    int4* unit_cand = nullptr;         // overflow scratch of the per-unit step kernel's candidate lists

    // kernel profiler: (kind, start, stop) event triples awaiting a read
    bool profiling = false;
    struct ProfRec { int kind; cudaEvent_t a, b; };
    std::vector<ProfRec> prof;
    std::vector<cudaEvent_t> ev_pool;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t copy_event = nullptr;
};

namespace skv {

// Launches `kernel` on `st` with programmatic stream serialization (PDL): the kernel may start
// while the previous kernel of the stream drains; it calls pdl_wait() before reading any input.
// pdl_enabled(): the score / select / attend kernels (opt-in, SKV_PDL=1); pdl_step_enabled(): the
// one-launch step kernel (default on, SKV_PDL=0 turns it off).
bool pdl_enabled();
bool pdl_step_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_if(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                          Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// ---- kernel launchers (each returns the cudaError_t of the launch) ----

// P1: sentence offsets for B prompts.  tokens [B][L]; off [B][Smax_cap+1]; S [B].
cudaError_t launch_segment(const int32_t* tokens, int B, int L, const int32_t* bset, int nb, int tau,
                           int32_t* off, int off_stride, int32_t* S, cudaStream_t st);

// P2: E = bf16(mean of member keys).  K [B][G][L][d]; off [B][Smax+1]; E [B][G][Smax][d].
cudaError_t launch_compress(const __nv_bfloat16* K, int B, int G, int L, int d, const int32_t* off,
                            int off_stride, const int32_t* S, int Smax, __nv_bfloat16* E, cudaStream_t st);

// D1: scores [B][G][Smax] of qt_g against every sentence embedding.
cudaError_t launch_score(const __nv_bfloat16* q, const float* Sq, const int32_t* cnt, const __nv_bfloat16* E,
                         const int32_t* S, int B, int G, int grp, int d, int Smax, float* scores,
                         cudaStream_t st);

// D2: budgeted selection + Q_s state update (Sq += q or reset).
cudaError_t launch_select(const float* scores, const int32_t* off, int off_stride, const int32_t* S, int B,
                          int G, int Smax, int tau, SelBufs sel, bool src_gathered, int32_t* out_ids,
                          int32_t* out_count, int32_t* out_tokens, cudaStream_t st);

// D3 + D4 with host residency: selected sentences also selected at the previous step are re-read
// from the previous HBM working-set slot, the others from the mapped pinned host store (PCIe); the
// staged rows are written through to the current slot; host bytes are added to *ledger.
cudaError_t launch_attend_host(const __nv_bfloat16* q, const __nv_bfloat16* Kh, const __nv_bfloat16* Vh, int L,
                               __nv_bfloat16* wsK, __nv_bfloat16* wsV, int B, int G, int grp, int d, SelBufs sel,
                               unsigned long long* ledger, QsState qs, float* out, cudaStream_t st);

// D3 + D4: split-K attention over the selected sentences' tokens (device residency).
cudaError_t launch_attend(const __nv_bfloat16* q, KvSrc kv, int B, int G, int grp, int d, SelBufs sel, QsState qs,
                          float* out, cudaStream_t st);

int attend_chunk_tokens(int d);

// ---- persistent per-layer kernel (decode_layer.cu): D1-D4 for every unit in one launch ----
struct LayerArgs {  // kernel parameter of layer_kernel
    // inputs / state (device residency)
    const __nv_bfloat16* q;        // [B][Hq][d]
    const int32_t* input_token;    // [B]
    const int32_t* bset;
    int nb;
    float* Sq;                     // [B][Hq][d]
    int32_t* cnt;                  // [B][G]
    const __nv_bfloat16* E;        // [B][G][Smax][d]
    const int32_t* S;              // [B]
    const int32_t* off;            // [B][off_stride]
    int off_stride;
    float* scores;                 // [B][G][Smax]
    SelBufs sel;
    KvSrc kv;
    float* out;                    // [B][Hq][d]
    int32_t* out_ids;              // optional [B][G][tau]
    int32_t* out_count;            // optional [B][G]
    int32_t* out_tokens;           // optional [B][G]
    // schedule
    const int2* items;             // (kind, unit | index << 16)
    int n_items;
    int B, G, Smax, tau;
    float scale_log2;
    // scratch (zeroed once; every launch returns it to zero)
    uint32_t* ticket;
    uint32_t* exit_count;
    uint32_t* score_done;          // [units]
    uint32_t* select_done;         // [units]
    uint32_t* attend_done;         // [units]
    float* part_ml;                // [units][n_att][8][2]
    float* part_o;                 // [units][n_att][8][D]
    int n_att;                     // ATTEND items per unit
    int4* cand;                    // [units][n_score_max][NL] (id, key, len, -) local candidates
    int32_t* cand_count;           // [units][n_score_max]
    int n_score_max;               // SCORE items of the unit with the most sentences
};

bool layer_enabled();
int layer_score_items(int d, int S_b);
int layer_attend_items(int tau);
int layer_item_sentences(int d);
std::vector<int2> layer_schedule(const std::vector<int>& S_host, int G, int d, int tau, int group);
size_t layer_smem_bytes(int d, int Smax, int tau);
cudaError_t launch_layer(const LayerArgs& a, int grp, int d, cudaStream_t st);


// D3 + D4 on tensor cores (mma.sync m16n8k16, decode_attend_mma.cu), both residencies; default
// (SKV_ATTEND=fma selects the fp32-FMA kernels above).
bool mma_enabled();
cudaError_t launch_attend_mma(const __nv_bfloat16* q, KvSrc kv, const __nv_bfloat16* Kh, const __nv_bfloat16* Vh,
                              int L, __nv_bfloat16* wsK, __nv_bfloat16* wsV, bool host, int B, int G, int grp, int d,
                              SelBufs sel, unsigned long long* ledger, QsState qs, float* out, cudaStream_t st);

// D2 + D3 + D4 fused (one cluster per unit), reading the scores of launch_score.  Opt-in
// (SKV_FUSED=1): on B200 the cluster-wide selection phases cost more than the separate select
// kernel (profiles/r01_notes.md).
bool fused_enabled();
bool fused_supported(int d, int grp, int Smax, int tau);
cudaError_t launch_fused_select_attend(const float* scores, const int32_t* off, int off_stride, const int32_t* S,
                                       int B, int G, int grp, int d, int Smax, int tau, const __nv_bfloat16* q,
                                       const int32_t* input_token, const int32_t* bset, int nb, float* Sq,
                                       int32_t* cnt, KvSrc kv, SelBufs sel, int32_t* out_ids, int32_t* out_count,
                                       int32_t* out_tokens, float* out, cudaStream_t st);

// ---- one launch per layer and step (decode_unit.cu): D1-D4 in one cluster per (b, g) unit ----
// Host residency (P3 + D3): the HBM working set of a unit is a page cache of `slots` pages of
// unit_page_tokens() context rows; pt maps a context page to its slot (-1 = not resident), own
// maps a slot to its page (-1 = empty), hand is the clock hand of the slot search.
struct HostCache {
    const __nv_bfloat16* Kh;       // mapped pinned host store [B][G][L][d] (nullptr: device residency)
    const __nv_bfloat16* Vh;
    __nv_bfloat16* wsK;            // [units][slots][page][d]
    __nv_bfloat16* wsV;
    int32_t* pt;                   // [units][pages]
    int32_t* own;                  // [units][slots]
    int32_t* hand;                 // [units]
    int slots, pages, L;
    unsigned long long* ledger;    // host bytes read (cumulative)
};
struct UnitArgs {
    const __nv_bfloat16* q;        // [B][Hq][d]
    const int32_t* input_token;    // [B]
    const int32_t* bset;
    int nb;
    float* Sq;                     // [B][Hq][d]
    int32_t* cnt;                  // [B][G]
    const __nv_bfloat16* E;        // [B][G][Smax][d]
    const int32_t* S;              // [B]
    const int32_t* off;            // [B][off_stride]
    int off_stride;
    int B, G, Smax;
    float* scores;                 // [B][G][Smax]
    SelBufs sel;
    KvSrc kv;                      // device residency: context K/V
    HostCache hc;                  // host residency (hc.Kh == nullptr in device residency)
    int4* cand;                    // [unit_cand_entries] overflow scratch of the candidate lists
    uint2* hint;                   // [units] selection band of the previous step (klo, khi ordered keys)
    int prefetch;                  // L2 prefetch of the previous step's selection
    const __nv_bfloat16* E_next;   // nullable: the next layer's E, prefetched into L2 while HBM idles
    float* out;                    // [B][Hq][d]
    int32_t* out_ids;              // optional [B][G][tau]
    int32_t* out_count;            // optional [B][G]
    int32_t* out_tokens;           // optional [B][G]
};
bool unit_enabled();
bool unit_supported(int d, int grp, int Smax, int tau, int slots);
int unit_page_tokens();
size_t unit_smem_bytes(int d, int tau);
size_t unit_cand_entries(int units);
cudaError_t launch_unit(const UnitArgs& a, int grp, int d, cudaStream_t st);

}  // namespace skv
