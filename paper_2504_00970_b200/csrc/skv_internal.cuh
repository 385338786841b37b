// skv_internal.cuh -- shared declarations of the SentenceKV sm_100a kernels and the runtime
// context behind the C ABI (include/sentencekv.h).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/sentencekv.h"
#include "mma_attend.cuh"

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
// NEXT-2 local segment / generated rows (Kg == nullptr: off).  Rows >= L of a layer's buckets are
// generated rows (row - L of the store); gstat[b] = {count, start of the current sentence, pending, overflow}.
// Also the NEXT-1 observation window (retention): its N rows are the `fixed` always-attended rows.
// Attended beyond the selection: store rows [0, fixed) and [gstat.start, gstat.count).
struct GenSrc {
    const __nv_bfloat16* Kg;       // [B][G][stride][d]
    const __nv_bfloat16* Vg;
    const int32_t* gstat;          // [B][4]
    int stride, L;
    int fixed;                     // always-attended rows at the start of the store
    int max_att;                   // upper bound of the attended rows beyond the selection (smem sizing)
};

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
    uint2* unit_hint = nullptr;        // [units] one-launch step kernel: band of the selection's crossing point
    int32_t* pc_pt = nullptr;          // host residency, one-launch kernel: page table [units][pages]
    int32_t* pc_own = nullptr;         // [units][slots]
    int32_t* pc_hand = nullptr;        // [units]
    int pc_pages = 0;
    int last_path = 0;                 // host residency: 1 = one-launch kernel (page cache), 2 = split kernels
    // NEXT-1 importance retention (cfg.obs_window > 0): the layer's retained pool and its buckets
    bool retained = false;
    int ret_m = 0;                     // pool tokens per sequence: min(floor(r*tau), L - N)
    __nv_bfloat16* PK = nullptr;       // [B][G][m][d] retained keys / values, token order (ctx-owned, HBM)
    __nv_bfloat16* PV = nullptr;
    float* alpha = nullptr;            // [B][L-N] token importance (Sec. 4.1)
    int32_t* keep = nullptr;           // [B][m]   retained token indices, ascending
    int32_t* roff = nullptr;           // [B][m+1] bucket offsets into the pool
    int32_t* rsid = nullptr;           // [B][m]   sentence id of each bucket
    int32_t* rS = nullptr;             // [B]      buckets (sentences with a retained token)
    size_t ret_bytes = 0;              // allocation key (B, G, m, L, N)
    // NEXT-2 local segment and growth (cfg.max_generated > 0)
    __nv_bfloat16* genK = nullptr;     // [B][G][max_gen][d] generated tokens' K / V
    __nv_bfloat16* genV = nullptr;
    int32_t* gstat = nullptr;          // [B][4]
    int32_t* goff = nullptr;           // [B][Smax+1] the prompt's offsets followed by completed generated sentences
    int32_t* gS = nullptr;             // [B] buckets
    int32_t* gsid = nullptr;           // retention + NEXT-2: [B][Smax] bucket -> sentence id (generated: S + k)
    int32_t* gS0 = nullptr;            // retention + NEXT-2: [B] retained buckets at prefill
    // NEXT-1 observation window, always attended with retention (reading A25)
    __nv_bfloat16* winK = nullptr;     // [B][G][N][d]
    __nv_bfloat16* winV = nullptr;
    int32_t* wstat = nullptr;          // [B][4] = {N, N, 0, 0}: no generated sentence in progress
    // SURVEY 8(e) fused all-gather epilogue (sentencekv_set_output_peers)
    OutPeers peers{};
    unsigned int* peer_local_flag = nullptr;  // this rank's arrival counter for the layer (peer memory)
    unsigned int* peer_target = nullptr;      // device: arrivals expected so far
    unsigned int peer_per_step = 0;           // world * units per rank
};

}  // namespace skv

struct skv_ctx {
    skv_config cfg{};
    int B = 0, G = 0, Hq = 0, grp = 0, d = 0, tau = 0;
    std::string err;
    skv_status sticky = SKV_OK;
    int64_t launches = 0;
    int band_log2 = 19;                // half-width of the step kernel's selection band (ordered-key units)

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
    int4* unit_cand = nullptr;         // overflow scratch of the per-unit step kernel's candidate lists
    int32_t* cap_dev = nullptr;        // NEXT-3 outlier split: per-prompt length cap [B]
    int32_t* seg_scratch = nullptr;    // P1: per-chunk last boundary and ends
    size_t seg_scratch_n = 0;
    float* ret_scratch = nullptr;      // NEXT-1 pass A partials + row stats
    size_t ret_scratch_n = 0;

    // kernel profiler: (kind, start, stop) event triples awaiting a read
    bool profiling = false;
    struct ProfRec { int kind; cudaEvent_t a, b; };
    std::vector<ProfRec> prof;
    std::vector<cudaEvent_t> ev_pool;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t copy_event = nullptr;
    bool after_prefill = false;        // a prefill kernel was the last launch of this context
};

namespace skv {

// Launches `kernel` on `st` with programmatic stream serialization (PDL): the kernel may start
// while the previous kernel of the stream drains; it calls pdl_wait() before reading any input.
// launch_pdl_if(false, ...) launches without the attribute (e.g. right after a prefill kernel
// whose writes the kernel reads before its pdl_wait()).
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
// ---- kernel launchers (each returns the cudaError_t of the launch) ----

// P1: sentence offsets for B prompts.  tokens [B][L]; off [B][Smax_cap+1]; S [B]; cap_b [B] or
// nullptr: a per-prompt length cap below tau (NEXT-3 outlier split).
cudaError_t launch_segment(const int32_t* tokens, int B, int L, const int32_t* bset, int nb, int tau,
                           int32_t* off, int off_stride, int32_t* S, const int32_t* cap_b, int32_t* scratch,
                           cudaStream_t st);
size_t segment_scratch_ints(int B, int L);  // scratch of launch_segment; bset must be sorted ascending

// ---- NEXT-3 / NEXT-4 bucket and ranking variants (variants.cu) ----
// outlier split threshold T = floor((L + n * sqrt(S * sum len^2 - L^2)) / S) per prompt (reading A27)
cudaError_t launch_outlier_cap(const int32_t* off, int off_stride, const int32_t* S, int B, double n, int32_t* cap,
                               cudaStream_t st);
// equal chunks (len = min(tau, ceil(L / S_b)), A26) or fixed pages (len = page > 0): off [B][stride], S [B]
cudaError_t launch_chunks(int B, int L, int tau, int page, int32_t* off, int off_stride, int32_t* S, cudaStream_t st);
// Quest page bounds: E [B][G][Smax][2][d] = (min, max) of each page's keys
cudaError_t launch_quest_meta(const __nv_bfloat16* K, int B, int G, int L, int d, int page, const int32_t* S, int Smax,
                              __nv_bfloat16* E, cudaStream_t st);
// Quest scores [B][G][Smax]: sum_h sum_j max(q_j mn_j, q_j mx_j), current query (reading A28)
cudaError_t launch_quest_score(const __nv_bfloat16* q, const __nv_bfloat16* E, const int32_t* S, int B, int G, int grp,
                               int d, int Smax, float* scores, cudaStream_t st);
// skip-and-continue fill on top of the prefix selection of launch_select (same outputs, rewritten)
cudaError_t launch_skip_fill(const float* scores, const int32_t* off, int off_stride, const int32_t* S, int B, int G,
                             int Smax, int tau, SelBufs sel, bool src_gathered, int32_t* out_ids, int32_t* out_count,
                             int32_t* out_tokens, const int32_t* sid, int sid_stride, cudaStream_t st);

// P2: E = bf16(mean of member keys).  K [B][G][L][d]; off [B][Smax+1]; E [B][G][Smax][d].
cudaError_t launch_compress(const __nv_bfloat16* K, int B, int G, int L, int d, const int32_t* off,
                            int off_stride, const int32_t* S, int Smax, __nv_bfloat16* E, cudaStream_t st);

// D1: scores [B][G][Smax] of qt_g against every sentence embedding.
cudaError_t launch_score(const __nv_bfloat16* q, const float* Sq, const int32_t* cnt, const __nv_bfloat16* E,
                         const int32_t* S, int B, int G, int grp, int d, int Smax, float* scores, int qmode,
                         cudaStream_t st);

// D2: budgeted selection + Q_s state update (Sq += q or reset).
cudaError_t launch_select(const float* scores, const int32_t* off, int off_stride, const int32_t* S, int B,
                          int G, int Smax, int tau, SelBufs sel, bool src_gathered, int32_t* out_ids,
                          int32_t* out_count, int32_t* out_tokens, const int32_t* sid, int sid_stride,
                          cudaStream_t st);

// D3 + D4 on tensor cores (mma.sync m16n8k16, decode_attend_mma.cu) over the selection of the
// last launch_select, both residencies.  Host residency: sentences also selected at the previous
// step are re-read from the previous HBM working-set slot, the others from the mapped pinned host
// store (PCIe); every row is written through to the current slot; host bytes are added to *ledger.
cudaError_t launch_attend_mma(const __nv_bfloat16* q, KvSrc kv, const __nv_bfloat16* Kh, const __nv_bfloat16* Vh,
                              int L, __nv_bfloat16* wsK, __nv_bfloat16* wsV, bool host, int B, int G, int grp, int d,
                              SelBufs sel, unsigned long long* ledger, QsState qs, float* out, GenSrc gen,
                              OutPeers peers, cudaStream_t st);

// SURVEY 8(e) fused gather: wait until `target` (advanced by `per_step` on the device each call)
// arrivals have been counted in *flag (acquire, system scope).
cudaError_t launch_wait_peers(const unsigned int* flag, unsigned int* target, unsigned int per_step, cudaStream_t st);

// NEXT-2 (local.cu): close the sentence that ended at the previous token into a bucket, append this
// token's k, v ([B][G][d]) to the generated store, advance the per-sequence state
cudaError_t launch_gen_append(const __nv_bfloat16* k, const __nv_bfloat16* v, __nv_bfloat16* Kg, __nv_bfloat16* Vg,
                              int max_gen, int32_t* gstat, int32_t* goff, int off_stride, int32_t* gS, int Smax,
                              __nv_bfloat16* E, const int32_t* input_token, const int32_t* bset, int nb, int B, int G,
                              int L, int d, int tau, int32_t* gsid, const int32_t* S_prompt, const int32_t* gS0,
                              cudaStream_t st);

// Opt-in dynamic shared memory of `func` on the current device (the attribute is per device
// context; cached per (device, function), thread-safe).
cudaError_t ensure_smem(const void* func, size_t smem);

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
    bool pdl;                      // launch with programmatic stream serialization
    int band_w;                    // half-width of the selection band (ordered-key units)
    float* out;                    // [B][Hq][d]
    int32_t* out_ids;              // optional [B][G][tau]
    int32_t* out_count;            // optional [B][G]
    int32_t* out_tokens;           // optional [B][G]
    const int32_t* sid;            // optional [B][sid_stride]: output ids = sid[b][selected bucket] (retention)
    int sid_stride;
    int qmode;                     // 0 = Eq. 2 mean query, 1 = current token's query (NEXT-3)
    GenSrc gen;                    // NEXT-2 local segment (gen.Kg == nullptr: off)
    OutPeers peers;                // 8(e) fused gather (peers.n == 0: off)
};
bool unit_supported(int d, int grp, int Smax, int tau, int slots, int pages, int local_att);
int unit_page_tokens();
size_t unit_smem_bytes(int d, int tau, int att);
size_t unit_cand_entries(int units);
cudaError_t launch_unit(const UnitArgs& a, int grp, int d, cudaStream_t st);

// ---- NEXT-1 importance-filtered retention at prefill (retain.cu) ----
struct RetainArgs {
    const __nv_bfloat16* q_window;  // [B][N][Hq][d] queries of the last N prompt tokens
    const __nv_bfloat16* K;         // [B][G][L][d]
    const __nv_bfloat16* V;
    int B, G, grp, d, L, N, m;      // m = retained tokens per sequence
    const int32_t* off;             // prompt sentence offsets [B][off_stride], S [B]
    int off_stride;
    const int32_t* S;
    float* alpha;                   // [B][L-N]
    float* scratch;                 // retain_scratch_floats(B, G, L, N, grp)
    int32_t* keep;                  // [B][m]
    int32_t* roff;                  // [B][m+1]
    int32_t* rsid;                  // [B][m]
    int32_t* rS;                    // [B]
    __nv_bfloat16* PK;              // [B][G][m][d]
    __nv_bfloat16* PV;
};
bool retain_supported(int d, int N, int grp);
size_t retain_scratch_floats(int B, int G, int L, int N, int grp);
cudaError_t launch_retain(const RetainArgs& a, cudaStream_t st);

}  // namespace skv
