// abi.cu -- skv_ctx runtime and the C ABI of include/sentencekv.h.
//
// Host-side responsibilities: argument validation (synchronous, state unchanged on error),
// ownership of device / pinned-host buffers, stream ordering, sticky CUDA errors.  Every step of
// the method runs in the kernels of prefill.cu, decode_select.cu and decode_attend.cu.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <vector>
#include <mutex>
#include <new>

#include "skv_internal.cuh"

#define SKV_API extern "C" __attribute__((visibility("default")))

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

skv_status fail(skv_ctx* ctx, skv_status st, const char* fmt, ...) __attribute__((format(printf, 3, 4)));
skv_status fail(skv_ctx* ctx, skv_status st, const char* fmt, ...) {
    if (ctx) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof(buf), fmt, ap);
        va_end(ap);
        ctx->err = buf;
    }
    return st;
}

skv_status cuda_fail(skv_ctx* ctx, cudaError_t e, const char* where) {
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        return fail(ctx, SKV_ERR_OUT_OF_MEMORY, "%s: %s", where, cudaGetErrorString(e));
    }
    ctx->sticky = SKV_ERR_CUDA;
    return fail(ctx, SKV_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define SKV_CUDA(ctx, expr)                                          \
    do {                                                             \
        cudaError_t e_ = (expr);                                     \
        if (e_ != cudaSuccess) return cuda_fail((ctx), e_, #expr);   \
    } while (0)

template <typename T>
cudaError_t dalloc(T** p, size_t n) {
    *p = nullptr;
    if (n == 0) return cudaSuccess;
    return cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T));
}

template <typename T>
void dfree(T*& p) {
    if (p) cudaFree((void*)p);
    p = nullptr;
}

void free_sel(skv::SelBufs& s) {
    dfree(s.ids);
    dfree(s.tokoff);
    dfree(s.src);
    dfree(s.count);
    dfree(s.parity);
}

void free_local(skv::LayerState& ls) {
    dfree(ls.gsid);
    dfree(ls.gS0);
    dfree(ls.genK);
    dfree(ls.genV);
    dfree(ls.gstat);
    dfree(ls.goff);
    dfree(ls.gS);
}

void free_layer_prompt(skv::LayerState& ls) {
    dfree(ls.E);
    dfree(ls.scores);
    free_sel(ls.sel);
    dfree(ls.wsK);
    dfree(ls.wsV);
    dfree(ls.unit_hint);
    dfree(ls.pc_pt);
    dfree(ls.pc_own);
    dfree(ls.pc_hand);
    free_local(ls);
}

void free_retention(skv::LayerState& ls) {
    dfree(ls.winK);
    dfree(ls.winV);
    dfree(ls.wstat);
    dfree(ls.PK);
    dfree(ls.PV);
    dfree(ls.alpha);
    dfree(ls.keep);
    dfree(ls.roff);
    dfree(ls.rsid);
    dfree(ls.rS);
    ls.ret_bytes = 0;
    ls.retained = false;
    ls.ret_m = 0;
}

void free_host_store(skv::LayerState& ls) {
    if (ls.Kh) cudaFreeHost(ls.Kh);
    if (ls.Vh) cudaFreeHost(ls.Vh);
    ls.Kh = ls.Vh = nullptr;
    ls.host_bytes = 0;
    ls.host_ready = false;
}

void free_prompt_buffers(skv_ctx* c) {
    for (auto& ls : c->layer) {
        free_layer_prompt(ls);
        ls.prefilled = false;
        ls.selected = false;
        ls.K = ls.V = nullptr;
    }
    dfree(c->off);
    c->Smax = 0;
    c->L = 0;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ---- kernel profiler: events bracketing each launch on its stream ----
cudaEvent_t prof_event(skv_ctx* c) {
    if (!c->ev_pool.empty()) {
        cudaEvent_t e = c->ev_pool.back();
        c->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

cudaEvent_t prof_begin(skv_ctx* c, cudaStream_t st) {
    if (!c->profiling) return nullptr;
    cudaEvent_t a = prof_event(c);
    cudaEventRecord(a, st);
    return a;
}

void prof_end(skv_ctx* c, int kind, cudaEvent_t a, cudaStream_t st) {
    if (!a) return;
    cudaEvent_t b = prof_event(c);
    cudaEventRecord(b, st);
    c->prof.push_back({kind, a, b});
}

}  // namespace

cudaError_t skv::ensure_smem(const void* func, size_t smem) {
    // cudaFuncSetAttribute is per device context: remember (device, function) -> bytes set
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    size_t& have = done[{dev, func}];
    if (smem <= have) return cudaSuccess;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (e == cudaSuccess) have = smem;
    return e;
}

SKV_API void sentencekv_config_default(skv_config* cfg) {
    if (!cfg) return;
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->semantic_factor = 2.0f;
    cfg->residency = SKV_KV_DEVICE;
}

SKV_API skv_status sentencekv_create(const skv_config* cfg_in, skv_ctx** out) {
    if (!cfg_in || !out) return SKV_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    skv_config cfg = *cfg_in;
    if (cfg.batch < 1 || cfg.layers < 1 || cfg.q_heads < 1 || cfg.kv_heads < 1 || cfg.head_dim < 1 ||
        cfg.max_context < 1 || cfg.token_budget < 1 || !(cfg.semantic_factor >= 1.0f) ||
        cfg.q_heads % cfg.kv_heads != 0 || (cfg.residency != SKV_KV_DEVICE && cfg.residency != SKV_KV_HOST))
        return SKV_ERR_INVALID_ARGUMENT;
    if (cfg.kv_head_count == 0) cfg.kv_head_count = cfg.kv_heads - cfg.kv_head_begin;
    if (cfg.batch_count == 0) cfg.batch_count = cfg.batch - cfg.batch_begin;
    if (cfg.kv_head_begin < 0 || cfg.kv_head_count < 1 || cfg.kv_head_begin + cfg.kv_head_count > cfg.kv_heads ||
        cfg.batch_begin < 0 || cfg.batch_count < 1 || cfg.batch_begin + cfg.batch_count > cfg.batch)
        return SKV_ERR_INVALID_ARGUMENT;
    const int grp = cfg.q_heads / cfg.kv_heads;
    if (cfg.obs_window < 0) return SKV_ERR_INVALID_ARGUMENT;
    // NEXT-3 / NEXT-4 modes
    if (cfg.bucket_mode < SKV_BUCKETS_SENTENCE || cfg.bucket_mode > SKV_BUCKETS_QUEST ||
        (cfg.bucket_mode == SKV_BUCKETS_QUEST && (cfg.chunk_size < 1 || cfg.chunk_size > cfg.token_budget)) ||
        !(cfg.outlier_n >= 0.0f) || (cfg.outlier_n > 0.0f && cfg.bucket_mode != SKV_BUCKETS_SENTENCE) ||
        (cfg.query_mode != SKV_QUERY_MEAN && cfg.query_mode != SKV_QUERY_CURRENT) ||
        (cfg.fill_mode != SKV_FILL_PREFIX && cfg.fill_mode != SKV_FILL_SKIP))
        return SKV_ERR_INVALID_ARGUMENT;
    if (cfg.obs_window > 0 && cfg.bucket_mode == SKV_BUCKETS_QUEST) return SKV_ERR_UNSUPPORTED;
    if (cfg.max_generated < 0) return SKV_ERR_INVALID_ARGUMENT;
    // NEXT-2 local segment: sentence / equal buckets (either residency; generated rows stay in HBM)
    if (cfg.max_generated > 0 && cfg.bucket_mode == SKV_BUCKETS_QUEST) return SKV_ERR_UNSUPPORTED;
    if ((cfg.head_dim != 64 && cfg.head_dim != 128) || (grp != 1 && grp != 2 && grp != 4 && grp != 8) ||
        (cfg.obs_window > 0 && !skv::retain_supported(cfg.head_dim, cfg.obs_window, grp)))
        return SKV_ERR_UNSUPPORTED;
    // host residency keeps the previous and the current selection in HBM: 2*tau <= floor(r*tau)
    if (cfg.residency == SKV_KV_HOST && !(cfg.semantic_factor >= 2.0f)) return SKV_ERR_INVALID_ARGUMENT;

    skv_ctx* c = new (std::nothrow) skv_ctx();
    if (!c) return SKV_ERR_OUT_OF_MEMORY;
    c->cfg = cfg;
    c->B = cfg.batch_count;
    c->G = cfg.kv_head_count;
    c->grp = grp;
    c->Hq = c->G * grp;
    c->d = cfg.head_dim;
    c->tau = cfg.token_budget;
    c->layer.resize(cfg.layers);
    c->S_host.assign(c->B, 0);

    DeviceGuard dg(cfg.device);
    cudaError_t e = cudaSuccess;
    for (auto& ls : c->layer) {
        if (e == cudaSuccess) e = dalloc(&ls.Sq, (size_t)c->B * c->Hq * c->d);
        if (e == cudaSuccess) e = dalloc(&ls.cnt, (size_t)c->B * c->G);
        if (e == cudaSuccess) e = cudaMemset(ls.Sq, 0, sizeof(float) * c->B * c->Hq * c->d);
        if (e == cudaSuccess) e = cudaMemset(ls.cnt, 0, sizeof(int32_t) * c->B * c->G);
    }
    if (e == cudaSuccess && cfg.residency == SKV_KV_HOST) {
        e = cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking);
        for (auto& ls : c->layer) {
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ls.offload_done, cudaEventDisableTiming);
            if (e == cudaSuccess) e = dalloc(&ls.ledger, 1);
            if (e == cudaSuccess) e = cudaMemset(ls.ledger, 0, sizeof(unsigned long long));
        }
    }
    if (e == cudaSuccess) e = dalloc(&c->S_dev, (size_t)c->B);
    if (e == cudaSuccess) e = dalloc(&c->bset, (size_t)skv::kMaxBoundary);
    if (e != cudaSuccess) {
        cudaGetLastError();
        sentencekv_destroy(c);
        return e == cudaErrorMemoryAllocation ? SKV_ERR_OUT_OF_MEMORY : SKV_ERR_CUDA;
    }
    *out = c;
    return SKV_OK;
}

SKV_API skv_status sentencekv_destroy(skv_ctx* c) {
    if (!c) return SKV_OK;
    DeviceGuard dg(c->cfg.device);
    cudaDeviceSynchronize();
    free_prompt_buffers(c);
    for (auto& ls : c->layer) {
        dfree(ls.Sq);
        dfree(ls.cnt);
        dfree(ls.ledger);
        dfree(ls.peer_target);
        free_host_store(ls);
        free_retention(ls);
        if (ls.offload_done) cudaEventDestroy(ls.offload_done);
    }
    dfree(c->S_dev);
    dfree(c->bset);
    dfree(c->unit_cand);
    dfree(c->ret_scratch);
    dfree(c->cap_dev);
    dfree(c->seg_scratch);
    for (auto& r : c->prof) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    if (c->copy_event) cudaEventDestroy(c->copy_event);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    delete c;
    return SKV_OK;
}

SKV_API const char* sentencekv_last_error(const skv_ctx* c) { return c ? c->err.c_str() : "null context"; }

SKV_API skv_status sentencekv_sync(skv_ctx* c) {
    if (!c) return SKV_ERR_INVALID_ARGUMENT;
    DeviceGuard dg(c->cfg.device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(c, e, "sentencekv_sync");
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(c, e, "sentencekv_sync");
    if (c->sticky == SKV_OK && c->cfg.max_generated > 0) {  // NEXT-2: a full generated store is a state error
        std::vector<int32_t> st(4 * c->B);
        for (size_t l = 0; l < c->layer.size(); ++l) {
            if (!c->layer[l].gstat || !c->layer[l].prefilled) continue;
            if (cudaMemcpy(st.data(), c->layer[l].gstat, sizeof(int32_t) * 4 * c->B, cudaMemcpyDeviceToHost) != cudaSuccess)
                return cuda_fail(c, cudaGetLastError(), "sentencekv_sync");
            for (int b = 0; b < c->B; ++b)
                if (st[4 * b + 3]) return fail(c, SKV_ERR_STATE, "layer %zu: more than max_generated = %d tokens appended",
                                               l, c->cfg.max_generated);
        }
    }
    return c->sticky;
}

// Host residency, one-launch kernel: pages of the HBM working set per unit, floor(r * tau) tokens.
static int cache_slots(const skv_ctx* c) {
    const long long cap = (long long)std::floor((double)c->cfg.semantic_factor * (double)c->tau);
    return (int)std::max(1LL, cap / skv::unit_page_tokens());
}

// What the decode of a layer ranks and attends: the prompt's sentences over the context K/V, or
// (NEXT-1 retention) the retained buckets over the layer's HBM pool.
struct LayerView {
    const int32_t* off;
    int off_stride;
    const int32_t* S;
    const __nv_bfloat16* K;
    const __nv_bfloat16* V;
    long long stride;      // K/V rows per (b, g) unit
    const int32_t* sid;    // bucket -> sentence id (retention), else nullptr
    int sid_stride;
    bool host;             // rows come from the host store through the HBM working set
    skv::GenSrc gen;       // NEXT-2 generated rows + local segment (gen.Kg == nullptr: off)
};
static LayerView layer_view(const skv_ctx* c, const skv::LayerState& ls) {
    const skv::GenSrc none{nullptr, nullptr, nullptr, 0, 0x7fffffff, 0, 0};  // no generated rows
    if (ls.retained && ls.genK)  // + NEXT-2: the store = the window, then the generated rows (A29)
        return {ls.goff, c->Smax + 1, ls.gS, ls.PK, ls.PV, ls.ret_m, ls.gsid, c->Smax, false,
                skv::GenSrc{ls.genK, ls.genV, ls.gstat, c->cfg.max_generated + c->cfg.obs_window, ls.ret_m, 0,
                            c->cfg.obs_window + c->tau}};
    if (ls.retained)  // the pool; rows >= m are the observation window's, always attended (A25)
        return {ls.roff, ls.ret_m + 1, ls.rS, ls.PK, ls.PV, ls.ret_m, ls.rsid, ls.ret_m, false,
                skv::GenSrc{ls.winK, ls.winV, ls.wstat, c->cfg.obs_window, ls.ret_m, c->cfg.obs_window,
                            c->cfg.obs_window}};
    if (ls.genK)  // host residency: context rows through the working set, generated rows in HBM
        return {ls.goff, c->Smax + 1, ls.gS, ls.K, ls.V, c->L, nullptr, 0, c->cfg.residency == SKV_KV_HOST,
                skv::GenSrc{ls.genK, ls.genV, ls.gstat, c->cfg.max_generated, c->L, 0, c->tau}};
    return {c->off, c->off_stride, c->S_dev, ls.K, ls.V, c->L, nullptr, 0, c->cfg.residency == SKV_KV_HOST, none};
}

// Empties the page cache of a layer (every page -> host).
static skv_status reset_page_cache(skv_ctx* c, skv::LayerState& ls, cudaStream_t st) {
    const size_t U = (size_t)c->B * c->G;
    SKV_CUDA(c, cudaMemsetAsync(ls.pc_pt, 0xff, sizeof(int32_t) * U * ls.pc_pages, st));
    SKV_CUDA(c, cudaMemsetAsync(ls.pc_own, 0xff, sizeof(int32_t) * U * cache_slots(c), st));
    SKV_CUDA(c, cudaMemsetAsync(ls.pc_hand, 0, sizeof(int32_t) * U, st));
    ls.last_path = 0;
    return SKV_OK;
}

// Host residency keeps a working set per path (split kernels: previous + current selection;
// one-launch kernel: page cache).  Switching paths on a layer forgets the other path's state:
// no previous selection (the split path has no hits, the page-cache plan nothing to fill).
static skv_status switch_host_path(skv_ctx* c, skv::LayerState& ls, int path, cudaStream_t st) {
    if (c->cfg.residency != SKV_KV_HOST || ls.last_path == path) {
        ls.last_path = path;
        return SKV_OK;
    }
    if (ls.last_path != 0) {
        SKV_CUDA(c, cudaMemsetAsync(ls.sel.count, 0, sizeof(int32_t) * 2 * c->B * c->G, st));
        if (path == 1) {
            skv_status s = reset_page_cache(c, ls, st);
            if (s != SKV_OK) return s;
        }
    }
    ls.last_path = path;
    return SKV_OK;
}

// (Re)allocates the sentence-dependent buffers of every layer for a prompt with capacity Smax.
static skv_status alloc_prompt_buffers(skv_ctx* c, int Smax) {
    const size_t B = c->B, G = c->G, d = c->d, tau = c->tau, U = B * G;
    for (auto& ls : c->layer) {
        // Quest pages keep (min, max) per page instead of one mean
        SKV_CUDA(c, dalloc(&ls.E, B * G * Smax * d * (c->cfg.bucket_mode == SKV_BUCKETS_QUEST ? 2 : 1)));
        SKV_CUDA(c, dalloc(&ls.scores, B * G * Smax));
        skv::SelBufs& sb = ls.sel;
        sb.units = (int)U;
        sb.tau = (int)tau;
        SKV_CUDA(c, dalloc(&sb.ids, 2 * U * tau));
        SKV_CUDA(c, dalloc(&sb.tokoff, 2 * U * (tau + 1)));
        SKV_CUDA(c, dalloc(&sb.src, 2 * U * tau));
        SKV_CUDA(c, dalloc(&sb.count, 2 * U));
        SKV_CUDA(c, dalloc(&sb.parity, U));
        if (c->cfg.residency == SKV_KV_HOST) {
            // split kernels: [U][2][tau] gathered rows; one-launch kernel: [U][slots][page] rows
            const size_t rows = std::max((size_t)2 * tau, (size_t)cache_slots(c) * skv::unit_page_tokens());
            SKV_CUDA(c, dalloc(&ls.wsK, U * rows * d));
            SKV_CUDA(c, dalloc(&ls.wsV, U * rows * d));
            const int P = skv::unit_page_tokens();
            ls.pc_pages = (c->cfg.max_context + P - 1) / P;
            SKV_CUDA(c, dalloc(&ls.pc_pt, U * (size_t)ls.pc_pages));
            SKV_CUDA(c, dalloc(&ls.pc_own, U * (size_t)cache_slots(c)));
            SKV_CUDA(c, dalloc(&ls.pc_hand, U));
        }
        SKV_CUDA(c, dalloc(&ls.unit_hint, U));
        if (c->cfg.max_generated > 0) {
            // the store holds the observation window first when retention is on (always attended)
            const size_t mg = (size_t)c->cfg.max_generated + (size_t)c->cfg.obs_window;
            SKV_CUDA(c, dalloc(&ls.genK, U * mg * d));
            SKV_CUDA(c, dalloc(&ls.genV, U * mg * d));
            SKV_CUDA(c, dalloc(&ls.gstat, B * 4));
            SKV_CUDA(c, dalloc(&ls.goff, B * (size_t)(Smax + 1)));
            SKV_CUDA(c, dalloc(&ls.gS, B));
            if (c->cfg.obs_window > 0) {
                SKV_CUDA(c, dalloc(&ls.gsid, B * (size_t)Smax));
                SKV_CUDA(c, dalloc(&ls.gS0, B));
            }
        }
    }
    dfree(c->unit_cand);
    SKV_CUDA(c, dalloc(&c->unit_cand, skv::unit_cand_entries((int)U)));
    c->Smax = Smax;
    return SKV_OK;
}

SKV_API skv_status sentencekv_prefill_compress(skv_ctx* c, int32_t layer, const int32_t* token_ids, int32_t L,
                                               const int32_t* boundary_ids, int32_t n_boundary, const void* K,
                                               const void* V, float semantic_factor, int32_t token_budget,
                                               const void* q_window, skv_stream_t stream_) {
    if (!c) return SKV_ERR_INVALID_ARGUMENT;
    if (c->sticky != SKV_OK) return c->sticky;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_);
    if (layer < 0 || layer >= c->cfg.layers) return fail(c, SKV_ERR_STATE, "layer %d out of range", layer);
    if (L < 1 || L > c->cfg.max_context) return fail(c, SKV_ERR_INVALID_ARGUMENT, "L=%d outside [1, %d]", L, c->cfg.max_context);
    if (!K || !V || !aligned16(K) || !aligned16(V))
        return fail(c, SKV_ERR_INVALID_ARGUMENT, "K/V must be non-NULL and 16-byte aligned");
    if (semantic_factor != c->cfg.semantic_factor || token_budget != c->tau)
        return fail(c, SKV_ERR_INVALID_ARGUMENT, "semantic_factor/token_budget differ from the context config");
    const int N = c->cfg.obs_window;
    if (q_window != nullptr && N < 1)
        return fail(c, SKV_ERR_INVALID_ARGUMENT, "q_window given but cfg.obs_window (N) is 0");
    if (N > 0 && (q_window == nullptr || !aligned16(q_window)))
        return fail(c, SKV_ERR_INVALID_ARGUMENT, "cfg.obs_window = %d needs the window queries (16-byte aligned)", N);
    if (N > 0 && L <= N) return fail(c, SKV_ERR_INVALID_ARGUMENT, "L=%d must exceed the observation window N=%d", L, N);
    const bool quest = c->cfg.bucket_mode == SKV_BUCKETS_QUEST;
    if (layer == 0) {
        if (!quest && !token_ids) return fail(c, SKV_ERR_INVALID_ARGUMENT, "token_ids is NULL");
        if ((!quest || boundary_ids) && (!boundary_ids || n_boundary < 1 || n_boundary > skv::kMaxBoundary))
            return fail(c, SKV_ERR_INVALID_ARGUMENT, "boundary set must hold 1..%d ids", skv::kMaxBoundary);
    } else if (c->L != L || !c->layer[0].prefilled) {
        return fail(c, SKV_ERR_STATE, "prefill of layer %d before layer 0 of a prompt of length %d", layer, L);
    }
    DeviceGuard dg(c->cfg.device);

    if (layer == 0) {
        // ---- new prompt: P1 segmentation (once; shared by all layers and heads) ----
        if (c->L != L || !c->off) {
            dfree(c->off);
            SKV_CUDA(c, dalloc(&c->off, (size_t)c->B * (L + 1)));
            c->L = L;
            c->off_stride = L + 1;
        }
        if (boundary_ids && n_boundary > 0) {
            // sorted (the segmentation kernels test membership by binary search); pageable source: the
            // copy is staged before the call returns
            std::vector<int32_t> sorted(boundary_ids, boundary_ids + n_boundary);
            std::sort(sorted.begin(), sorted.end());
            SKV_CUDA(c, cudaMemcpyAsync(c->bset, sorted.data(), sizeof(int32_t) * n_boundary, cudaMemcpyHostToDevice, st));
            c->n_bset = n_boundary;
        } else {  // Quest without a boundary set: no input token resets Q_s (Quest does not use it)
            c->n_bset = 0;
        }
        const size_t need = skv::segment_scratch_ints(c->B, L);
        if (c->seg_scratch_n < need) {  // (allocated outside the profiled region)
            dfree(c->seg_scratch);
            c->seg_scratch_n = 0;
            SKV_CUDA(c, dalloc(&c->seg_scratch, need));
            c->seg_scratch_n = need;
        }
        if (c->cfg.outlier_n > 0.0f && !c->cap_dev) SKV_CUDA(c, dalloc(&c->cap_dev, (size_t)c->B));
        cudaEvent_t pa = prof_begin(c, st);
        if (quest) {  // NEXT-4: fixed pages of chunk_size tokens
            SKV_CUDA(c, skv::launch_chunks(c->B, L, c->tau, c->cfg.chunk_size, c->off, c->off_stride, c->S_dev, st));
            c->launches += 1;
        } else {
            SKV_CUDA(c, skv::launch_segment(token_ids, c->B, L, c->bset, n_boundary, c->tau, c->off, c->off_stride,
                                            c->S_dev, nullptr, c->seg_scratch, st));
            c->launches += 3;
            if (c->cfg.outlier_n > 0.0f) {  // NEXT-3 outlier split: re-segment under the per-prompt cap T
                SKV_CUDA(c, skv::launch_outlier_cap(c->off, c->off_stride, c->S_dev, c->B, (double)c->cfg.outlier_n,
                                                    c->cap_dev, st));
                SKV_CUDA(c, skv::launch_segment(token_ids, c->B, L, c->bset, n_boundary, c->tau, c->off,
                                                c->off_stride, c->S_dev, c->cap_dev, c->seg_scratch, st));
                c->launches += 4;
            } else if (c->cfg.bucket_mode == SKV_BUCKETS_EQUAL) {  // NEXT-3 equal chunks, as many as sentences
                SKV_CUDA(c, skv::launch_chunks(c->B, L, c->tau, 0, c->off, c->off_stride, c->S_dev, st));
                c->launches += 1;
            }
        }
        prof_end(c, SKV_K_SEGMENT, pa, st);
        SKV_CUDA(c, cudaMemcpyAsync(c->S_host.data(), c->S_dev, sizeof(int32_t) * c->B, cudaMemcpyDeviceToHost, st));
        SKV_CUDA(c, cudaStreamSynchronize(st));
        int Smax = 1;
        for (int b = 0; b < c->B; ++b) Smax = c->S_host[b] > Smax ? c->S_host[b] : Smax;
        Smax += c->cfg.max_generated;  // NEXT-2: room for every sentence the decode may add
        if (Smax > c->Smax || !c->layer[0].E) {
            for (auto& ls : c->layer) free_layer_prompt(ls);
            skv_status s = alloc_prompt_buffers(c, Smax);
            if (s != SKV_OK) return s;
        }
        for (auto& ls : c->layer) {
            ls.prefilled = false;
            ls.selected = false;
            // no previous selection (empty slot 0, parity 0): the host gather misses everything at the
            // first step
            SKV_CUDA(c, cudaMemsetAsync(ls.sel.count, 0, sizeof(int32_t) * 2 * c->B * c->G, st));
            SKV_CUDA(c, cudaMemsetAsync(ls.sel.parity, 0, sizeof(int32_t) * c->B * c->G, st));
            SKV_CUDA(c, cudaMemsetAsync(ls.Sq, 0, sizeof(float) * c->B * c->Hq * c->d, st));
            SKV_CUDA(c, cudaMemsetAsync(ls.cnt, 0, sizeof(int32_t) * c->B * c->G, st));
            // no band yet (klo = 0, khi = max: everything is in the band)
            SKV_CUDA(c, cudaMemsetAsync(ls.unit_hint, 0xff, sizeof(uint2) * c->B * c->G, st));
            SKV_CUDA(c, cudaMemset2DAsync(ls.unit_hint, sizeof(uint2), 0, sizeof(uint32_t), (size_t)c->B * c->G, st));
            if (c->cfg.residency == SKV_KV_HOST) {
                skv_status rs = reset_page_cache(c, ls, st);
                if (rs != SKV_OK) return rs;
            }
        }
    }

    skv::LayerState& ls = c->layer[layer];
    const auto* Kb = static_cast<const __nv_bfloat16*>(K);
    const auto* Vb = static_cast<const __nv_bfloat16*>(V);
    const bool host = c->cfg.residency == SKV_KV_HOST;
    size_t store_elems = (size_t)c->B * c->G * L * c->d;  // P3: what goes to the host store
    const __nv_bfloat16 *srcK = Kb, *srcV = Vb;
    if (N > 0) {
        // ---- NEXT-1: alpha, global top-floor(r*tau), retained pool + buckets (retain.cu), then Eq. 1
        // over the retained tokens of every sentence (Alg. 1 lines 4-7)
        const long long k = (long long)std::floor((double)c->cfg.semantic_factor * (double)c->tau);
        const int m = (int)std::min<long long>(k, (long long)(L - N));
        const size_t key = ((size_t)m << 32) ^ (size_t)(L - N);
        if (ls.ret_bytes != key || !ls.PK) {
            free_retention(ls);
            const size_t U = (size_t)c->B * c->G;
            SKV_CUDA(c, dalloc(&ls.PK, U * m * c->d));
            SKV_CUDA(c, dalloc(&ls.PV, U * m * c->d));
            SKV_CUDA(c, dalloc(&ls.alpha, (size_t)c->B * (L - N)));
            SKV_CUDA(c, dalloc(&ls.keep, (size_t)c->B * m));
            SKV_CUDA(c, dalloc(&ls.roff, (size_t)c->B * (m + 1)));
            SKV_CUDA(c, dalloc(&ls.rsid, (size_t)c->B * m));
            SKV_CUDA(c, dalloc(&ls.rS, (size_t)c->B));
            SKV_CUDA(c, dalloc(&ls.winK, U * N * c->d));
            SKV_CUDA(c, dalloc(&ls.winV, U * N * c->d));
            SKV_CUDA(c, dalloc(&ls.wstat, (size_t)c->B * 4));
            {
                std::vector<int32_t> ws(4 * c->B, 0);
                for (int b = 0; b < c->B; ++b) ws[4 * b] = ws[4 * b + 1] = N;
                SKV_CUDA(c, cudaMemcpy(ls.wstat, ws.data(), sizeof(int32_t) * 4 * c->B, cudaMemcpyHostToDevice));
            }
            ls.ret_bytes = key;
        }
        const size_t need = skv::retain_scratch_floats(c->B, c->G, L, N, c->grp);
        if (c->ret_scratch_n < need) {
            dfree(c->ret_scratch);
    dfree(c->cap_dev);
    dfree(c->seg_scratch);
            c->ret_scratch_n = 0;
            SKV_CUDA(c, dalloc(&c->ret_scratch, need));
            c->ret_scratch_n = need;
        }
        skv::RetainArgs ra{static_cast<const __nv_bfloat16*>(q_window), Kb, Vb, c->B, c->G, c->grp, c->d, L, N, m,
                           c->off, c->off_stride, c->S_dev, ls.alpha, c->ret_scratch, ls.keep, ls.roff, ls.rsid, ls.rS,
                           ls.PK, ls.PV};
        // the observation window's K/V rows [L-N, L): attended by every decode step (reading A25)
        SKV_CUDA(c, cudaMemcpy2DAsync(ls.winK, sizeof(__nv_bfloat16) * N * c->d, Kb + (size_t)(L - N) * c->d,
                                      sizeof(__nv_bfloat16) * L * c->d, sizeof(__nv_bfloat16) * N * c->d,
                                      (size_t)c->B * c->G, cudaMemcpyDeviceToDevice, st));
        SKV_CUDA(c, cudaMemcpy2DAsync(ls.winV, sizeof(__nv_bfloat16) * N * c->d, Vb + (size_t)(L - N) * c->d,
                                      sizeof(__nv_bfloat16) * L * c->d, sizeof(__nv_bfloat16) * N * c->d,
                                      (size_t)c->B * c->G, cudaMemcpyDeviceToDevice, st));
        cudaEvent_t pr = prof_begin(c, st);
        SKV_CUDA(c, skv::launch_retain(ra, st));
        prof_end(c, SKV_K_RETAIN, pr, st);
        c->launches += 5;
        cudaEvent_t pa = prof_begin(c, st);
        SKV_CUDA(c, skv::launch_compress(ls.PK, c->B, c->G, m, c->d, ls.roff, m + 1, ls.rS, c->Smax, ls.E, st));
        prof_end(c, SKV_K_COMPRESS, pa, st);
        c->launches += 1;
        ls.retained = true;
        ls.ret_m = m;
        store_elems = (size_t)c->B * c->G * m * c->d;  // the paper offloads the retained tokens (Alg. 1 l.7)
        srcK = ls.PK;
        srcV = ls.PV;
    } else {
        // ---- P2: Eq. 1 sentence embeddings of this layer (Quest: the pages' min / max keys) ----
        cudaEvent_t pa = prof_begin(c, st);
        if (quest)
            SKV_CUDA(c, skv::launch_quest_meta(Kb, c->B, c->G, L, c->d, c->cfg.chunk_size, c->S_dev, c->Smax, ls.E, st));
        else
            SKV_CUDA(c, skv::launch_compress(Kb, c->B, c->G, L, c->d, c->off, c->off_stride, c->S_dev, c->Smax, ls.E, st));
        prof_end(c, SKV_K_COMPRESS, pa, st);
        c->launches += 1;
        ls.retained = false;
    }
    if (host) {
        // P3: this layer's K/V (full, or the retained pool) -> ctx-owned pinned, mapped host memory, on
        // the copy stream
        const size_t bytes = sizeof(__nv_bfloat16) * store_elems;
        if (ls.host_bytes != bytes) {
            free_host_store(ls);
            void *hk = nullptr, *hv = nullptr;
            if (cudaHostAlloc(&hk, bytes, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
                cudaHostAlloc(&hv, bytes, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
                cudaGetLastError();
                if (hk) cudaFreeHost(hk);
                return fail(c, SKV_ERR_OUT_OF_MEMORY, "pinned host store of %zu bytes for layer %d", 2 * bytes, layer);
            }
            ls.Kh = static_cast<__nv_bfloat16*>(hk);
            ls.Vh = static_cast<__nv_bfloat16*>(hv);
            ls.host_bytes = bytes;
        }
        if (!c->copy_event) SKV_CUDA(c, cudaEventCreateWithFlags(&c->copy_event, cudaEventDisableTiming));
        SKV_CUDA(c, cudaEventRecord(c->copy_event, st));
        SKV_CUDA(c, cudaStreamWaitEvent(c->copy_stream, c->copy_event, 0));
        cudaEvent_t po = prof_begin(c, c->copy_stream);
        SKV_CUDA(c, cudaMemcpyAsync(ls.Kh, srcK, bytes, cudaMemcpyDeviceToHost, c->copy_stream));
        SKV_CUDA(c, cudaMemcpyAsync(ls.Vh, srcV, bytes, cudaMemcpyDeviceToHost, c->copy_stream));
        prof_end(c, SKV_K_OFFLOAD, po, c->copy_stream);
        SKV_CUDA(c, cudaEventRecord(ls.offload_done, c->copy_stream));
        ls.host_ready = false;
        ls.K = ls.V = nullptr;  // the caller may free its K/V after sentencekv_sync
        if (layer == 0)
            for (auto& l2 : c->layer) SKV_CUDA(c, cudaMemsetAsync(l2.ledger, 0, sizeof(unsigned long long), st));
    } else if (N > 0) {
        ls.K = ls.V = nullptr;  // the ctx keeps its own pool
    } else {
        ls.K = Kb;  // device residency: borrowed until the next prefill or destroy
        ls.V = Vb;
    }
    if (c->cfg.max_generated > 0 && ls.retained) {
        // NEXT-1 + NEXT-2 (reading A29): the buckets start as the retained buckets (and their sentence
        // ids); the store starts with the observation window's rows, which are the local segment when
        // decoding starts (attended every step, and part of the first generated bucket once the first
        // generated sentence ends); no generated token yet
        const int m = ls.ret_m;
        const size_t cap = (size_t)c->cfg.max_generated + N;
        SKV_CUDA(c, cudaMemcpy2DAsync(ls.goff, sizeof(int32_t) * (c->Smax + 1), ls.roff, sizeof(int32_t) * (m + 1),
                                      sizeof(int32_t) * std::min(m + 1, c->Smax + 1), c->B, cudaMemcpyDeviceToDevice, st));
        SKV_CUDA(c, cudaMemcpy2DAsync(ls.gsid, sizeof(int32_t) * c->Smax, ls.rsid, sizeof(int32_t) * m,
                                      sizeof(int32_t) * std::min(m, c->Smax), c->B, cudaMemcpyDeviceToDevice, st));
        SKV_CUDA(c, cudaMemcpyAsync(ls.gS, ls.rS, sizeof(int32_t) * c->B, cudaMemcpyDeviceToDevice, st));
        SKV_CUDA(c, cudaMemcpyAsync(ls.gS0, ls.rS, sizeof(int32_t) * c->B, cudaMemcpyDeviceToDevice, st));
        SKV_CUDA(c, cudaMemcpy2DAsync(ls.genK, sizeof(__nv_bfloat16) * cap * c->d, ls.winK,
                                      sizeof(__nv_bfloat16) * N * c->d, sizeof(__nv_bfloat16) * N * c->d,
                                      (size_t)c->B * c->G, cudaMemcpyDeviceToDevice, st));
        SKV_CUDA(c, cudaMemcpy2DAsync(ls.genV, sizeof(__nv_bfloat16) * cap * c->d, ls.winV,
                                      sizeof(__nv_bfloat16) * N * c->d, sizeof(__nv_bfloat16) * N * c->d,
                                      (size_t)c->B * c->G, cudaMemcpyDeviceToDevice, st));
        // the window rows are the local segment when decoding starts: {count N, sentence start 0}
        std::vector<int32_t> gs(4 * (size_t)c->B, 0);
        for (int b = 0; b < c->B; ++b) gs[4 * (size_t)b] = N;
        SKV_CUDA(c, cudaMemcpyAsync(ls.gstat, gs.data(), sizeof(int32_t) * gs.size(), cudaMemcpyHostToDevice, st));
    } else if (c->cfg.max_generated > 0) {
        // NEXT-2: the layer's buckets start as the prompt's sentences; no generated token yet
        SKV_CUDA(c, cudaMemcpy2DAsync(ls.goff, sizeof(int32_t) * (c->Smax + 1), c->off, sizeof(int32_t) * c->off_stride,
                                      sizeof(int32_t) * (std::min(c->off_stride, c->Smax + 1)), c->B,
                                      cudaMemcpyDeviceToDevice, st));
        SKV_CUDA(c, cudaMemcpyAsync(ls.gS, c->S_dev, sizeof(int32_t) * c->B, cudaMemcpyDeviceToDevice, st));
        SKV_CUDA(c, cudaMemsetAsync(ls.gstat, 0, sizeof(int32_t) * 4 * c->B, st));
    }
    ls.prefilled = true;
    ls.selected = false;
    c->after_prefill = true;
    return SKV_OK;
}

SKV_API skv_status sentencekv_decode_select(skv_ctx* c, int32_t layer, const void* q, const int32_t* input_token,
                                            int32_t* sel_ids, int32_t* sel_count, int32_t* sel_tokens,
                                            skv_stream_t stream_) {
    if (!c) return SKV_ERR_INVALID_ARGUMENT;
    if (c->sticky != SKV_OK) return c->sticky;
    if (layer < 0 || layer >= c->cfg.layers) return fail(c, SKV_ERR_STATE, "layer %d out of range", layer);
    skv::LayerState& ls = c->layer[layer];
    if (!ls.prefilled) return fail(c, SKV_ERR_STATE, "decode_select before prefill of layer %d", layer);
    if (!q || !input_token) return fail(c, SKV_ERR_INVALID_ARGUMENT, "q / input_token is NULL");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_);
    DeviceGuard dg(c->cfg.device);
    const auto* qb = static_cast<const __nv_bfloat16*>(q);
    const LayerView v = layer_view(c, ls);
    if (v.host) {
        skv_status ps = switch_host_path(c, ls, 2, st);
        if (ps != SKV_OK) return ps;
    }
    cudaEvent_t pa = prof_begin(c, st);
    if (c->cfg.bucket_mode == SKV_BUCKETS_QUEST)
        SKV_CUDA(c, skv::launch_quest_score(qb, ls.E, v.S, c->B, c->G, c->grp, c->d, c->Smax, ls.scores, st));
    else
        SKV_CUDA(c, skv::launch_score(qb, ls.Sq, ls.cnt, ls.E, v.S, c->B, c->G, c->grp, c->d, c->Smax, ls.scores,
                                      c->cfg.query_mode, st));
    prof_end(c, SKV_K_SCORE, pa, st);
    pa = prof_begin(c, st);
    SKV_CUDA(c, skv::launch_select(ls.scores, v.off, v.off_stride, v.S, c->B, c->G, c->Smax, c->tau, ls.sel, false,
                                   sel_ids, sel_count, sel_tokens, v.sid, v.sid_stride, st));
    c->launches += 2;
    if (c->cfg.fill_mode == SKV_FILL_SKIP) {  // NEXT-3 skip-and-continue on top of the prefix
        SKV_CUDA(c, skv::launch_skip_fill(ls.scores, v.off, v.off_stride, v.S, c->B, c->G, c->Smax, c->tau, ls.sel,
                                          false, sel_ids, sel_count, sel_tokens, v.sid, v.sid_stride, st));
        c->launches += 1;
    }
    prof_end(c, SKV_K_SELECT, pa, st);
    ls.selected = true;
    ls.input_token = input_token;
    return SKV_OK;
}

SKV_API skv_status sentencekv_decode_step(skv_ctx* c, int32_t layer, const void* q, const int32_t* input_token,
                                          float* out, int32_t* sel_ids, int32_t* sel_count, int32_t* sel_tokens,
                                          skv_stream_t stream_) {
    if (!c) return SKV_ERR_INVALID_ARGUMENT;
    if (c->sticky != SKV_OK) return c->sticky;
    if (layer < 0 || layer >= c->cfg.layers) return fail(c, SKV_ERR_STATE, "layer %d out of range", layer);
    skv::LayerState& ls = c->layer[layer];
    if (!ls.prefilled) return fail(c, SKV_ERR_STATE, "decode_step before prefill of layer %d", layer);
    if (!q || !input_token || !out) return fail(c, SKV_ERR_INVALID_ARGUMENT, "q / input_token / out is NULL");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_);
    DeviceGuard dg(c->cfg.device);
    const auto* qb = static_cast<const __nv_bfloat16*>(q);
    const LayerView v = layer_view(c, ls);
    const bool host = v.host;
    const bool unit_path = c->cfg.bucket_mode != SKV_BUCKETS_QUEST && c->cfg.fill_mode == SKV_FILL_PREFIX;
    if (unit_path && skv::unit_supported(c->d, c->grp, c->Smax, c->tau, host ? cache_slots(c) : 0,
                                         host ? ls.pc_pages : 0, v.gen.Kg ? v.gen.max_att : 0)) {
        // default: one launch per layer, one thread-block cluster per (b, g) unit (decode_unit.cu)
        skv::UnitArgs a{};
        if (host) {
            if (!ls.host_ready) {  // first decode of the layer after its prefill: the offload must be done
                SKV_CUDA(c, cudaEventSynchronize(ls.offload_done));
                ls.host_ready = true;
            }
            skv_status ps = switch_host_path(c, ls, 1, st);
            if (ps != SKV_OK) return ps;
            a.hc = skv::HostCache{ls.Kh, ls.Vh, ls.wsK, ls.wsV, ls.pc_pt, ls.pc_own, ls.pc_hand, cache_slots(c),
                                  ls.pc_pages, c->L, ls.ledger};
        }
        a.q = qb;
        a.input_token = input_token;
        a.bset = c->bset;
        a.nb = c->n_bset;
        a.Sq = ls.Sq;
        a.cnt = ls.cnt;
        a.E = ls.E;
        a.S = v.S;
        a.off = v.off;
        a.off_stride = v.off_stride;
        a.sid = v.sid;
        a.sid_stride = v.sid_stride;
        a.qmode = c->cfg.query_mode;
        a.gen = v.gen;
        a.peers = ls.peers;
        a.B = c->B;
        a.G = c->G;
        a.Smax = c->Smax;
        a.scores = ls.scores;
        a.sel = ls.sel;
        a.kv = skv::KvSrc{v.K, v.V, v.stride, 0};
        a.cand = c->unit_cand;
        a.hint = ls.unit_hint;
        a.band_w = 1 << c->band_log2;
        // the step kernel reads prefill outputs (S, offsets, E) before its programmatic-launch wait:
        // never overlap it with a prefill kernel
        a.pdl = !c->after_prefill;
        c->after_prefill = false;
        a.out = out;
        a.out_ids = sel_ids;
        a.out_count = sel_count;
        a.out_tokens = sel_tokens;
        cudaEvent_t pa = prof_begin(c, st);
        SKV_CUDA(c, skv::launch_unit(a, c->grp, c->d, st));
        prof_end(c, SKV_K_STEP, pa, st);
        c->launches += 1;
        ls.selected = true;
        ls.input_token = input_token;
        return SKV_OK;
    }
    // Quest pages, skip-and-continue fill, or the capacity fallback (Smax > 16384 sentences or a
    // selection too large for the step kernel's shared memory): the kernels of the split calls
    skv_status s = sentencekv_decode_select(c, layer, q, input_token, sel_ids, sel_count, sel_tokens, stream_);
    if (s != SKV_OK) return s;
    return sentencekv_decode_attend(c, layer, q, out, stream_);
}

SKV_API skv_status sentencekv_decode_append(skv_ctx* c, int32_t layer, const void* k, const void* v,
                                            const int32_t* input_token, skv_stream_t stream_) {
    if (!c) return SKV_ERR_INVALID_ARGUMENT;
    if (c->sticky != SKV_OK) return c->sticky;
    if (c->cfg.max_generated < 1) return fail(c, SKV_ERR_STATE, "decode_append needs cfg.max_generated > 0");
    if (layer < 0 || layer >= c->cfg.layers) return fail(c, SKV_ERR_STATE, "layer %d out of range", layer);
    skv::LayerState& ls = c->layer[layer];
    if (!ls.prefilled || !ls.genK) return fail(c, SKV_ERR_STATE, "decode_append before prefill of layer %d", layer);
    if (!k || !v || !input_token || !aligned16(k) || !aligned16(v))
        return fail(c, SKV_ERR_INVALID_ARGUMENT, "k / v (16-byte aligned) / input_token is NULL");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_);
    DeviceGuard dg(c->cfg.device);
    cudaEvent_t pa = prof_begin(c, st);
    const bool ret = ls.retained;
    SKV_CUDA(c, skv::launch_gen_append(static_cast<const __nv_bfloat16*>(k), static_cast<const __nv_bfloat16*>(v),
                                       ls.genK, ls.genV, c->cfg.max_generated + (ret ? c->cfg.obs_window : 0), ls.gstat,
                                       ls.goff, c->Smax + 1, ls.gS, c->Smax, ls.E, input_token, c->bset, c->n_bset, c->B,
                                       c->G, ret ? ls.ret_m : c->L, c->d, c->tau, ret ? ls.gsid : nullptr,
                                       ret ? c->S_dev : nullptr, ret ? ls.gS0 : nullptr, st));
    prof_end(c, SKV_K_APPEND, pa, st);
    c->launches += 2;
    return SKV_OK;
}

SKV_API skv_status sentencekv_set_output_peers(skv_ctx* c, int32_t layer, int32_t world, int32_t rank,
                                               float* const* peer_out, uint32_t* const* peer_flag) {
    if (!c) return SKV_ERR_INVALID_ARGUMENT;
    if (layer < 0 || layer >= c->cfg.layers) return fail(c, SKV_ERR_STATE, "layer %d out of range", layer);
    skv::LayerState& ls = c->layer[layer];
    if (world == 0 || !peer_out) {  // back to the caller's collective
        ls.peers = skv::OutPeers{};
        ls.peer_local_flag = nullptr;
        return SKV_OK;
    }
    if (world < 1 || world > skv::kMaxPeers || rank < 0 || rank >= world || !peer_flag)
        return fail(c, SKV_ERR_INVALID_ARGUMENT, "world must be 1..%d with rank < world and both pointer arrays",
                    skv::kMaxPeers);
    for (int p = 0; p < world; ++p)
        if (!peer_out[p] || !peer_flag[p] || !aligned16(peer_out[p]))
            return fail(c, SKV_ERR_INVALID_ARGUMENT, "peer %d: NULL or unaligned pointer", p);
    DeviceGuard dg(c->cfg.device);
    if (!ls.peer_target) {
        SKV_CUDA(c, dalloc(&ls.peer_target, 1));
    }
    SKV_CUDA(c, cudaMemset(ls.peer_target, 0, sizeof(unsigned int)));
    skv::OutPeers pp{};
    const size_t slot = (size_t)c->B * c->Hq * c->d;  // one rank's [B][Hq_loc][d] outputs
    for (int p = 0; p < world; ++p) {
        pp.out[p] = peer_out[p] + (size_t)rank * slot;
        pp.flag[p] = reinterpret_cast<unsigned int*>(peer_flag[p]);
    }
    pp.n = world;
    ls.peers = pp;
    ls.peer_local_flag = reinterpret_cast<unsigned int*>(peer_flag[rank]);
    ls.peer_per_step = (unsigned int)world * (unsigned int)(c->B * c->G);
    return SKV_OK;
}

SKV_API skv_status sentencekv_wait_outputs(skv_ctx* c, int32_t layer, skv_stream_t stream_) {
    if (!c) return SKV_ERR_INVALID_ARGUMENT;
    if (c->sticky != SKV_OK) return c->sticky;
    if (layer < 0 || layer >= c->cfg.layers) return fail(c, SKV_ERR_STATE, "layer %d out of range", layer);
    skv::LayerState& ls = c->layer[layer];
    if (!ls.peer_local_flag) return fail(c, SKV_ERR_STATE, "layer %d has no output peers", layer);
    DeviceGuard dg(c->cfg.device);
    SKV_CUDA(c, skv::launch_wait_peers(ls.peer_local_flag, ls.peer_target, ls.peer_per_step,
                                       reinterpret_cast<cudaStream_t>(stream_)));
    c->launches += 1;
    return SKV_OK;
}

SKV_API skv_status sentencekv_decode_attend(skv_ctx* c, int32_t layer, const void* q, float* out,
                                            skv_stream_t stream_) {
    if (!c) return SKV_ERR_INVALID_ARGUMENT;
    if (c->sticky != SKV_OK) return c->sticky;
    if (layer < 0 || layer >= c->cfg.layers) return fail(c, SKV_ERR_STATE, "layer %d out of range", layer);
    skv::LayerState& ls = c->layer[layer];
    if (!ls.prefilled || !ls.selected)
        return fail(c, SKV_ERR_STATE, "decode_attend of layer %d before its prefill and decode_select", layer);
    if (!q || !out) return fail(c, SKV_ERR_INVALID_ARGUMENT, "q / out is NULL");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_);
    DeviceGuard dg(c->cfg.device);
    const auto* qb = static_cast<const __nv_bfloat16*>(q);
    const skv::QsState qs{ls.input_token, c->bset, c->n_bset, ls.Sq, ls.cnt};
    const LayerView v = layer_view(c, ls);
    cudaEvent_t pa = nullptr;
    if (v.host) {
        if (!ls.host_ready) {  // first decode of the layer after its prefill: the offload must be done
            SKV_CUDA(c, cudaEventSynchronize(ls.offload_done));
            ls.host_ready = true;
        }
        pa = prof_begin(c, st);
        SKV_CUDA(c, skv::launch_attend_mma(qb, skv::KvSrc{ls.wsK, ls.wsV, 0, 0}, ls.Kh, ls.Vh, c->L, ls.wsK, ls.wsV,
                                           true, c->B, c->G, c->grp, c->d, ls.sel, ls.ledger, qs, out, v.gen, ls.peers,
                                           st));
    } else {
        pa = prof_begin(c, st);
        const skv::KvSrc kv{v.K, v.V, v.stride, 0};
        SKV_CUDA(c, skv::launch_attend_mma(qb, kv, nullptr, nullptr, (int)v.stride, nullptr, nullptr, false, c->B, c->G,
                                           c->grp, c->d, ls.sel, nullptr, qs, out, v.gen, ls.peers, st));
    }
    prof_end(c, SKV_K_ATTEND, pa, st);
    c->launches += 1;
    return SKV_OK;
}

// ------------------------------------------------------------------------------ introspection

SKV_API skv_status sentencekv_sentence_counts(skv_ctx* c, int32_t* S_out) {
    if (!c || !S_out) return SKV_ERR_INVALID_ARGUMENT;
    if (!c->layer[0].prefilled) return fail(c, SKV_ERR_STATE, "no prompt");
    std::memcpy(S_out, c->S_host.data(), sizeof(int32_t) * c->B);
    return SKV_OK;
}

SKV_API int32_t sentencekv_sentence_capacity(const skv_ctx* c) { return c ? c->Smax : 0; }

SKV_API skv_status sentencekv_copy_offsets(skv_ctx* c, int32_t* off_out, skv_stream_t stream_) {
    if (!c || !off_out) return SKV_ERR_INVALID_ARGUMENT;
    if (!c->layer[0].prefilled) return fail(c, SKV_ERR_STATE, "no prompt");
    DeviceGuard dg(c->cfg.device);
    SKV_CUDA(c, cudaMemcpy2DAsync(off_out, sizeof(int32_t) * (c->Smax + 1), c->off, sizeof(int32_t) * c->off_stride,
                                  sizeof(int32_t) * (c->Smax + 1), c->B, cudaMemcpyDeviceToDevice,
                                  reinterpret_cast<cudaStream_t>(stream_)));
    return SKV_OK;
}

SKV_API skv_status sentencekv_copy_embeddings(skv_ctx* c, int32_t layer, void* E_out, skv_stream_t stream_) {
    if (!c || !E_out) return SKV_ERR_INVALID_ARGUMENT;
    if (layer < 0 || layer >= c->cfg.layers || !c->layer[layer].prefilled) return fail(c, SKV_ERR_STATE, "layer not prefilled");
    DeviceGuard dg(c->cfg.device);
    SKV_CUDA(c, cudaMemcpyAsync(E_out, c->layer[layer].E,
                                sizeof(__nv_bfloat16) * c->B * c->G * c->Smax * c->d *
                                    (c->cfg.bucket_mode == SKV_BUCKETS_QUEST ? 2 : 1),
                                cudaMemcpyDeviceToDevice, reinterpret_cast<cudaStream_t>(stream_)));
    return SKV_OK;
}

SKV_API skv_status sentencekv_copy_scores(skv_ctx* c, int32_t layer, float* out, skv_stream_t stream_) {
    if (!c || !out) return SKV_ERR_INVALID_ARGUMENT;
    if (layer < 0 || layer >= c->cfg.layers || !c->layer[layer].selected) return fail(c, SKV_ERR_STATE, "layer not selected");
    DeviceGuard dg(c->cfg.device);
    SKV_CUDA(c, cudaMemcpyAsync(out, c->layer[layer].scores, sizeof(float) * c->B * c->G * c->Smax,
                                cudaMemcpyDeviceToDevice, reinterpret_cast<cudaStream_t>(stream_)));
    return SKV_OK;
}

SKV_API int64_t sentencekv_launch_count(const skv_ctx* c) { return c ? c->launches : 0; }

SKV_API int32_t sentencekv_retained_tokens(const skv_ctx* c, int32_t layer) {
    if (!c || layer < 0 || layer >= c->cfg.layers || !c->layer[layer].retained) return 0;
    return c->layer[layer].ret_m;
}

SKV_API skv_status sentencekv_copy_importance(skv_ctx* c, int32_t layer, float* alpha_out, skv_stream_t stream_) {
    if (!c || !alpha_out) return SKV_ERR_INVALID_ARGUMENT;
    if (layer < 0 || layer >= c->cfg.layers || !c->layer[layer].retained)
        return fail(c, SKV_ERR_STATE, "layer %d has no retention", layer);
    DeviceGuard dg(c->cfg.device);
    SKV_CUDA(c, cudaMemcpyAsync(alpha_out, c->layer[layer].alpha, sizeof(float) * c->B * (c->L - c->cfg.obs_window),
                                cudaMemcpyDeviceToDevice, reinterpret_cast<cudaStream_t>(stream_)));
    return SKV_OK;
}

SKV_API skv_status sentencekv_copy_retained(skv_ctx* c, int32_t layer, int32_t* keep_out, int32_t* off_out,
                                            int32_t* sid_out, int32_t* S_out, skv_stream_t stream_) {
    if (!c) return SKV_ERR_INVALID_ARGUMENT;
    if (layer < 0 || layer >= c->cfg.layers || !c->layer[layer].retained)
        return fail(c, SKV_ERR_STATE, "layer %d has no retention", layer);
    DeviceGuard dg(c->cfg.device);
    const skv::LayerState& ls = c->layer[layer];
    const size_t m = ls.ret_m;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_);
    if (keep_out) SKV_CUDA(c, cudaMemcpyAsync(keep_out, ls.keep, sizeof(int32_t) * c->B * m, cudaMemcpyDeviceToDevice, st));
    if (off_out) SKV_CUDA(c, cudaMemcpyAsync(off_out, ls.roff, sizeof(int32_t) * c->B * (m + 1), cudaMemcpyDeviceToDevice, st));
    if (sid_out) SKV_CUDA(c, cudaMemcpyAsync(sid_out, ls.rsid, sizeof(int32_t) * c->B * m, cudaMemcpyDeviceToDevice, st));
    if (S_out) SKV_CUDA(c, cudaMemcpyAsync(S_out, ls.rS, sizeof(int32_t) * c->B, cudaMemcpyDeviceToDevice, st));
    return SKV_OK;
}

SKV_API skv_status sentencekv_host_fetch_bytes(skv_ctx* c, int32_t layer, uint64_t* bytes_out) {
    if (!c || !bytes_out) return SKV_ERR_INVALID_ARGUMENT;
    if (layer < 0 || layer >= c->cfg.layers) return fail(c, SKV_ERR_STATE, "layer %d out of range", layer);
    if (c->cfg.residency != SKV_KV_HOST) {
        *bytes_out = 0;
        return SKV_OK;
    }
    DeviceGuard dg(c->cfg.device);
    unsigned long long v = 0;
    SKV_CUDA(c, cudaMemcpy(&v, c->layer[layer].ledger, sizeof(v), cudaMemcpyDeviceToHost));
    *bytes_out = v;
    return SKV_OK;
}

SKV_API skv_status sentencekv_set_band_log2(skv_ctx* c, int32_t log2) {
    if (!c || log2 < 0 || log2 > 29) return SKV_ERR_INVALID_ARGUMENT;
    c->band_log2 = log2;
    return SKV_OK;
}

SKV_API skv_status sentencekv_set_profiling(skv_ctx* c, int32_t on) {
    if (!c) return SKV_ERR_INVALID_ARGUMENT;
    c->profiling = on != 0;
    if (c->profiling) {  // events created up front: creating one between two records would be timed
        DeviceGuard dg(c->cfg.device);
        while (c->ev_pool.size() < 256) {
            cudaEvent_t e = nullptr;
            if (cudaEventCreate(&e) != cudaSuccess) break;
            c->ev_pool.push_back(e);
        }
    }
    return SKV_OK;
}

SKV_API skv_status sentencekv_profile_read(skv_ctx* c, double* ms_out, int64_t* n_out) {
    if (!c || !ms_out || !n_out) return SKV_ERR_INVALID_ARGUMENT;
    DeviceGuard dg(c->cfg.device);
    for (auto& r : c->prof) {
        SKV_CUDA(c, cudaEventSynchronize(r.b));
        float ms = 0.0f;
        SKV_CUDA(c, cudaEventElapsedTime(&ms, r.a, r.b));
        ms_out[r.kind] += ms;
        n_out[r.kind] += 1;
        c->ev_pool.push_back(r.a);
        c->ev_pool.push_back(r.b);
    }
    c->prof.clear();
    return SKV_OK;
}
