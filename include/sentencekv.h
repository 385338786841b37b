/*
 * sentencekv.h -- C ABI of the SentenceKV hot path on B200 (sm_100a).
 *
 * Library: paper_2504_00970_b200/libsentencekv.so (built by __graft_entry__.build()).
 * Paper:   "SentenceKV" (arXiv 2504.00970); "P:<n>" = line n of PAPER.md, with the section,
 *          equation or algorithm line it falls in.  Readings A1..A23 are listed in DESIGN.md.
 *
 * Conventions for every entry point:
 *   - Plain C types only; no C++ exception crosses the boundary; every call returns skv_status.
 *   - "device" pointers are CUDA device pointers on cfg.device; "host" pointers are ordinary
 *     host memory.  The caller owns every pointer it passes in.
 *   - All GPU work is enqueued on the given cudaStream_t (NULL = legacy default stream);
 *     results are valid once that stream has completed the call's work.
 *   - Argument errors are reported synchronously (SKV_ERR_INVALID_ARGUMENT / _STATE /
 *     _UNSUPPORTED) and leave the context unchanged.  CUDA launch or asynchronous errors are
 *     sticky: returned as SKV_ERR_CUDA by the call that sees them or by sentencekv_sync(), with
 *     text from sentencekv_last_error().
 *   - Decode entry points do no allocation, so a whole decode step (all layers) can be captured
 *     into a CUDA graph.  The only host synchronisation on the decode path: in SKV_KV_HOST, the
 *     FIRST decode call of a layer after its prefill waits (cudaEventSynchronize) for that layer's
 *     P3 offload copy; run one eager decode step before capturing.
 *   - One context per host thread (single writer).  Contexts are independent.
 *   - Tensor layouts are row-major, innermost dimension last; bf16 = IEEE bfloat16 bits.
 *   - Multi-GPU: each rank creates one context over its shard (kv_head_begin/count,
 *     batch_begin/count); every pointer passed is shard-local ([batch_count][...]).  The
 *     all-gather of per-head outputs is done by the caller (torch.distributed, NCCL).
 */
#ifndef SENTENCEKV_H
#define SENTENCEKV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* skv_stream_t; /* == cudaStream_t */
typedef struct skv_ctx skv_ctx;

typedef enum {
    SKV_OK = 0,
    SKV_ERR_INVALID_ARGUMENT = 1, /* NULL pointer, non-positive size, Hq % G != 0, shard out of range,
                                     tau < 1, r < 1, L < 1 or L > max_context, n_boundary < 1 or > 64,
                                     K/V not 16-byte aligned, semantic_factor/token_budget != cfg, an unknown
                                     bucket/query/fill mode, a Quest page outside [1, tau], outlier_n < 0 or
                                     outlier_n > 0 with non-sentence buckets */
    SKV_ERR_STATE = 2,            /* layer out of range, decode before that layer's prefill, prefill of
                                     layer > 0 before layer 0 of the same prompt */
    SKV_ERR_UNSUPPORTED = 3,      /* head_dim not in {64, 128}; grp not in {1, 2, 4, 8}; retention with Quest
                                     pages; obs_window N > 0
                                     with N * grp not a multiple of 16 or above 256 (the window rows of
                                     one KV head form the N side of one tensor-core MMA) */
    SKV_ERR_CUDA = 4,             /* CUDA launch / asynchronous failure (sticky; see last_error) */
    SKV_ERR_OUT_OF_MEMORY = 5     /* device or pinned-host allocation failed */
} skv_status;

typedef enum {
    SKV_KV_DEVICE = 0, /* K/V stay in HBM, borrowed from the caller (kept until next prefill/destroy) */
    SKV_KV_HOST = 1    /* P3: full K/V offloaded to ctx-owned pinned, mapped host memory.  D3
                          (P:448): the HBM working set of each (sequence, layer, KV head) holds
                          floor(r*tau) tokens (needs r >= 2).  sentencekv_decode_step: a page cache of
                          16-token pages (rows resident in HBM are read there, the others from host
                          memory over PCIe and written through).  decode_select + decode_attend: the
                          previous and the current selection (2*tau rows); sentences selected again are
                          re-read from HBM, the others fetched from host memory. */
} skv_residency;

/* what a bucket is, which query ranks them, how the budget is filled */
typedef enum {
    SKV_BUCKETS_SENTENCE = 0, /* sentences at the boundary tokens (P1) */
    SKV_BUCKETS_EQUAL = 1,    /* NEXT-3 equal-size chunks, as many as the prompt has sentences, each
                                 min(tau, ceil(L / S)) tokens (Sec. 6.1 ablation; reading A26) */
    SKV_BUCKETS_QUEST = 2     /* NEXT-4 Quest: fixed pages of chunk_size tokens ranked by the bound
                                 sum_h sum_j max(q_j min_j, q_j max_j) of the current query over each
                                 page's per-dimension min / max keys (App. Quest; reading A28) */
} skv_bucket_mode;
typedef enum {
    SKV_QUERY_MEAN = 0,       /* Eq. 2 mean of the sentence cache Q_s */
    SKV_QUERY_CURRENT = 1     /* NEXT-3 current token's query (Sec. 6.2 ablation) */
} skv_query_mode;
typedef enum {
    SKV_FILL_PREFIX = 0,      /* maximal prefix of the ranking that fits tau (reading A13) */
    SKV_FILL_SKIP = 1         /* NEXT-3 skip-and-continue: walk the whole ranking, take what still fits */
} skv_fill_mode;

typedef struct {
    int32_t batch;           /* B: sequences in the global batch */
    int32_t layers;          /* M: transformer layers */
    int32_t q_heads;         /* Hq: query heads (global) */
    int32_t kv_heads;        /* G: KV heads (global); grp = Hq / G query heads share one KV head */
    int32_t head_dim;        /* d in {64, 128} */
    int32_t max_context;     /* L_max: largest prompt length accepted */
    int32_t token_budget;    /* tau >= 1: retrieved tokens per (sequence, layer, KV head) (A15) */
    float semantic_factor;   /* r >= 1; host residency needs r >= 2: its HBM working set holds
                                the previous and the current selection, 2*tau <= floor(r*tau) tokens per
                                (sequence, layer, KV head) (A19, A20) */
    int32_t obs_window;      /* N: observation-window size of the importance retention (SURVEY 8(f)
                                NEXT-1, see sentencekv_prefill_compress); 0 = no retention (every token of a
                                sentence is kept, reading A6) */
    int32_t residency;       /* skv_residency */
    int32_t device;          /* CUDA device ordinal */
    int32_t kv_head_begin;   /* this rank's KV-head shard [begin, begin+count); 0, G = all */
    int32_t kv_head_count;
    int32_t batch_begin;     /* this rank's batch shard [begin, begin+count); 0, B = all */
    int32_t batch_count;
    int32_t bucket_mode;     /* skv_bucket_mode (default SKV_BUCKETS_SENTENCE) */
    int32_t chunk_size;      /* SKV_BUCKETS_QUEST: page size in tokens, 1 <= chunk_size <= tau (16, 32 in the paper) */
    float outlier_n;         /* NEXT-3 outlier split (App. "Effect of Sentence Length"; reading A27):
                                > 0 cuts every sentence longer than T = floor(mean + outlier_n * std) of the
                                prompt's sentence lengths into pieces of T tokens; 0 = off (SENTENCE buckets only) */
    int32_t query_mode;      /* skv_query_mode (default SKV_QUERY_MEAN; Quest always ranks by the current query) */
    int32_t fill_mode;       /* skv_fill_mode (default SKV_FILL_PREFIX) */
    int32_t max_generated;   /* NEXT-2 (reading A29): > 0 keeps a local segment and grows the context -- up to
                                this many generated tokens per (sequence, layer) appended with
                                sentencekv_decode_append; 0 = off.  Either residency (the generated
                                rows stay in HBM; in host residency the context rows go through the
                                working set), without Quest pages (else UNSUPPORTED).  With retention
                                (obs_window > 0) the buckets start as the retained buckets and the
                                observation window's rows start the local segment (they close with the
                                first generated sentence). */
} skv_config;

/* Fills cfg with defaults (shard = everything, device residency, r = 2, obs_window = 0). */
void sentencekv_config_default(skv_config* cfg);

/* Creates a context.  Allocates the per-layer query-cache state (Sq fp32 [M][B][Hq][d]) on
 * cfg->device.  Sentence-dependent buffers are sized at the first prefill of a prompt.
 * Errors: INVALID_ARGUMENT (see skv_status), UNSUPPORTED, OUT_OF_MEMORY, CUDA. */
skv_status sentencekv_create(const skv_config* cfg, skv_ctx** out);

/* Frees everything the context owns.  Synchronises the device first.  NULL is a no-op. */
skv_status sentencekv_destroy(skv_ctx* ctx);

/* Text of the last error of this context ("" if none).  Valid until the next call. */
const char* sentencekv_last_error(const skv_ctx* ctx);

/* Waits for all work of this context and surfaces asynchronous CUDA errors. */
skv_status sentencekv_sync(skv_ctx* ctx);

/*
 * Prefill, one call per layer (Alg. 1 lines 2-8).
 *   P1 (layer 0 only): split each prompt into sentence buckets at the boundary tokens
 *      (Sec. 4.1; readings A1-A5: membership in boundary_ids, the boundary token
 *      ends its sentence, no merging, trailing tokens form the last sentence, tau-cap).
 *      Calling layer 0 starts a new prompt: it resets every layer's sentence query cache and
 *      invalidates every layer's embeddings.  This call synchronises the stream once to learn
 *      the sentence counts (prefill is not on the per-token path).
 *   P2: sentence embeddings kbar_{s,g} = bf16(mean of the sentence's keys) (Eq. 1, P:402-405;
 *      A6, A7, A23), kept in HBM (ctx-owned, [B][G][S_max][d] bf16 per layer).
 *   P3 (SKV_KV_HOST): full K and V copied to ctx-owned pinned host memory (A19)
 *      on an internal copy stream ordered after the caller's stream; the caller may free K/V
 *      after sentencekv_sync().  SKV_KV_DEVICE: the ctx borrows K and V (no copy).
 *
 * token_ids     device int32 [batch_count][L]  (layer 0 only; ignored for layer > 0 and for Quest pages,
 *               may then be NULL).  NEXT-3 / NEXT-4 bucket variants replace P1 by equal chunks, outlier-split
 *               sentences or Quest pages (see skv_config.bucket_mode / outlier_n); Quest replaces P2's
 *               Eq. 1 means by the pages' min / max keys.
 * L             prompt length, 1 <= L <= max_context; identical for every layer of a prompt
 * boundary_ids  host int32 [n_boundary], 1 <= n_boundary <= 64: the punctuation token-id set
 *               (layer 0 only; ignored for layer > 0)
 * K, V          device bf16 [batch_count][kv_head_count][L][d], contiguous, 16-byte aligned
 * semantic_factor, token_budget  must equal cfg values (checked; the paper's REQUIRE line, Alg. 1
 *               "Prompt tokens, token budget tau, semantic keeping factor r, observation window
 *               size N")
 * q_window      device bf16 [batch_count][N][kv_head_count*grp][d], 16-byte aligned, or NULL: queries of
 *               the last N = cfg.obs_window prompt tokens (the observation window, Sec. 4.1).
 *               cfg.obs_window == 0: must be NULL (no retention, reading A6; non-NULL is
 *               INVALID_ARGUMENT).  cfg.obs_window = N > 0: required, and L > N (else INVALID_ARGUMENT);
 *               the layer is prefilled with importance-filtered retention:
 *                 alpha_j = sum over window tokens w and all query heads h of the softmax, over w's
 *                   causal prefix, of q_{w,h} . k_j / sqrt(d), for j < L - N (reading A21;
 *                   two tcgen05 tensor-core passes, fp32 -- within the tolerance of reading A24);
 *                 the global top m = min(floor(r * tau), L - N) tokens by alpha are retained (ties ->
 *                   lowest index), the rest discarded;
 *                 each sentence keeps its retained tokens as a bucket (sentences with none are dropped,
 *                   reading A25); Eq. 1 runs over the retained tokens only;
 *                 the retained K/V form a ctx-owned pool in HBM ([B][G][m][d], token order) that every
 *                 decode call of the layer ranks and attends (the HBM working set of floor(r*tau)
 *                 tokens holds all of it); the N window tokens' K/V are kept too and attended by every
 *                 decode step besides the selection, uncharged (reading A25); K/V are not borrowed:
 *                 the caller may free them after sentencekv_sync.  SKV_KV_HOST: P3 offloads the pool, not the full K/V (Alg. 1 l.7,
 *                 P:580 "Offload a small subset (r*tau) of tokens to CPU").
 *               Decode outputs (sel_ids) stay the prompt's sentence ids; sel_tokens count retained
 *               tokens.  Introspection: sentencekv_copy_importance / sentencekv_copy_retained.
 */
skv_status sentencekv_prefill_compress(skv_ctx* ctx, int32_t layer, const int32_t* token_ids, int32_t L,
                                       const int32_t* boundary_ids, int32_t n_boundary, const void* K,
                                       const void* V, float semantic_factor, int32_t token_budget,
                                       const void* q_window, skv_stream_t stream);

/*
 * Decode, per layer per step: D1 + D2 (Alg. 1 lines 14-17).
 *   D1: append q_t to the layer's sentence query cache and form qbar (Eq. 2; A10),
 *       group query qt_g = sum of the group's qbar_h (A9), similarity qt_g^T kbar_{s,g} for every
 *       sentence (A23 canonical fp32).  If input_token[b] is a boundary id, the cache
 *       of sequence b is reset after this step (A11).  The cache update itself (append or
 *       reset) is applied by the decode_attend of the same layer and step, which must follow.
 *   D2: per (sequence, KV head): the maximal prefix of the ranking (score desc, index asc)
 *       whose token count fits tau (A13, A14); result kept in the ctx for decode_attend.
 *
 * q            device bf16 [batch_count][kv_head_count*grp][d]: this step's query (as cached)
 * input_token  device int32 [batch_count]: the token whose query this is; it must stay valid until the
 *              decode_attend of the same layer has executed (that call applies the Eq. 2 update)
 * sel_ids      device int32 [batch_count][kv_head_count][tau] or NULL: selected sentence ids,
 *              ascending, tail filled with -1
 * sel_count    device int32 [batch_count][kv_head_count] or NULL: number of selected sentences
 * sel_tokens   device int32 [batch_count][kv_head_count] or NULL: selected tokens (<= tau)
 */
skv_status sentencekv_decode_select(skv_ctx* ctx, int32_t layer, const void* q, const int32_t* input_token,
                                    int32_t* sel_ids, int32_t* sel_count, int32_t* sel_tokens,
                                    skv_stream_t stream);

/*
 * Decode, per layer per step: D3 + D4 (Alg. 1 lines 18-19) over the selection made
 * by the last decode_select of the same layer.
 *   D3: gather the selected sentences' K/V rows (contiguous runs) into shared memory with bulk
 *       async copies (device residency: from the caller's K/V in HBM; host residency: sentences
 *       also selected at the previous step from the HBM working set, the others from the pinned
 *       host store over PCIe, the staged rows written through to the working set).
 *   D4: O = softmax(q K_sel^T / sqrt(d)) V_sel (Eq. 3; A16-A18), split-K
 *       flash-decode with fp32 online softmax, combined in-kernel.
 *
 * q    device bf16 [batch_count][kv_head_count*grp][d]
 * out  device fp32 [batch_count][kv_head_count*grp][d]
 */
skv_status sentencekv_decode_attend(skv_ctx* ctx, int32_t layer, const void* q, float* out,
                                    skv_stream_t stream);

/*
 * Decode, per layer per step: D1 + D2 + D3 + D4 in one call (Alg. 1 lines 14-19).
 * Same selection as sentencekv_decode_select followed by sentencekv_decode_attend (same arithmetic,
 * bit-identical ids; O within the same tolerance).  Runs as ONE kernel launch per call: a
 * thread-block cluster of 8 CTAs per (sequence, KV head) scores its sentences, selects, gathers
 * and attends (decode_unit.cu).  When the prompt exceeds that kernel's capacity (more than 16384
 * sentences per sequence, or a budget whose selection tables do not fit its shared memory) the
 * call runs the score, select and attend kernels of the two split calls instead (same results).
 *
 * q, input_token  as in sentencekv_decode_select
 * out             device fp32 [batch_count][kv_head_count*grp][d]
 * sel_ids, sel_count, sel_tokens  optional outputs, as in sentencekv_decode_select (NULL allowed)
 */
skv_status sentencekv_decode_step(skv_ctx* ctx, int32_t layer, const void* q, const int32_t* input_token,
                                  float* out, int32_t* sel_ids, int32_t* sel_count, int32_t* sel_tokens,
                                  skv_stream_t stream);

/*
 * NEXT-2 (cfg.max_generated > 0; "After generating the next token, we append its query to Q_s
 * and repeat"; reading A29), per layer per step, BEFORE that step's decode_select / decode_step:
 *   - if the sentence being generated ended at the previous step's token (a boundary input, A11, or
 *     tau tokens long, A5), it becomes a retrievable bucket of the layer: Eq. 1 mean of its keys
 *     appended to the layer's embeddings, its rows appended to the layer's bucket offsets (rows
 *     >= L are generated rows; sel_ids >= the prompt's sentence count name generated sentences --
 *     the k-th one is sel_id S + k, S the prompt's sentence count, with or without retention);
 *   - this step's k, v are appended to the generated store; the tokens of the sentence being
 *     generated (this one included) form the local segment, which decode_attend / decode_step attend
 *     in addition to the selection, not charged to tau.
 * k, v         device bf16 [batch_count][kv_head_count][d], 16-byte aligned: this token's key / value
 * input_token  device int32 [batch_count]: as in decode_select (the same array may be passed)
 * More than max_generated appends: the token is dropped and sentencekv_sync returns STATE.
 */
skv_status sentencekv_decode_append(skv_ctx* ctx, int32_t layer, const void* k, const void* v,
                                    const int32_t* input_token, skv_stream_t stream);

/*
 * Multi-GPU: the per-layer all-gather of the per-head outputs fused into the attention
 * epilogue.  After this call, every decode_attend / decode_step of `layer` also stores its outputs
 * into slot `rank` of every peer's gather buffer and, once the unit's outputs are in, adds 1 to every
 * peer's arrival counter (release, system scope).
 * peer_out   host array [world] of device pointers, peer-accessible from this device (e.g. torch
 *            symmetric memory over NVLink): rank p's buffer fp32 [world][batch_count][kv_head_count*grp][d]
 *            (the rank-major layout of an all-gather; all ranks hold equal shards)
 * peer_flag  host array [world] of device pointers to uint32 arrival counters, zero at the first step
 * world = 0 or peer_out == NULL turns it off (the caller's collective).  world <= 8.
 */
skv_status sentencekv_set_output_peers(skv_ctx* ctx, int32_t layer, int32_t world, int32_t rank, float* const* peer_out,
                                       uint32_t* const* peer_flag);

/* Enqueues on `stream` a wait until every rank's outputs of this step's `layer` are in this rank's buffer
 * (world x units arrivals more than at the previous call; acquire, system scope).  CUDA-graph capturable. */
skv_status sentencekv_wait_outputs(skv_ctx* ctx, int32_t layer, skv_stream_t stream);

/* ---- introspection (tests, bench; not on the per-token path) ---- */

/* Sentence counts of the current prompt: S_out host int32 [batch_count]. */
skv_status sentencekv_sentence_counts(skv_ctx* ctx, int32_t* S_out);

/* Capacity S_max of the per-(b,g) sentence arrays of the current prompt (>= every S_b). */
int32_t sentencekv_sentence_capacity(const skv_ctx* ctx);

/* Sentence offsets of the current prompt: off_out device int32 [batch_count][S_max+1]
 * (row b holds off[0..S_b], rest unspecified).  Enqueued on stream. */
skv_status sentencekv_copy_offsets(skv_ctx* ctx, int32_t* off_out, skv_stream_t stream);

/* Layer embeddings: E_out device bf16 [batch_count][kv_head_count][S_max][d]. */
skv_status sentencekv_copy_embeddings(skv_ctx* ctx, int32_t layer, void* E_out, skv_stream_t stream);

/* Scores of the last decode_select of the layer: device fp32 [batch_count][kv_head_count][S_max]. */
skv_status sentencekv_copy_scores(skv_ctx* ctx, int32_t layer, float* scores_out, skv_stream_t stream);

/* Host residency ledger: bytes of K/V fetched from host memory by the decode steps of `layer`
 * since its prompt's prefill (synchronous).  0 in device residency. */
skv_status sentencekv_host_fetch_bytes(skv_ctx* ctx, int32_t layer, uint64_t* bytes_out);

/* NEXT-1 retention of `layer` (cfg.obs_window > 0): m = retained tokens per sequence (0 if the layer
 * has no retention). */
int32_t sentencekv_retained_tokens(const skv_ctx* ctx, int32_t layer);

/* alpha_out device fp32 [batch_count][L - N]: the token importance of the layer's prefill. */
skv_status sentencekv_copy_importance(skv_ctx* ctx, int32_t layer, float* alpha_out, skv_stream_t stream);

/* The layer's retained pool (each output nullable, device int32): keep_out [batch_count][m] retained token
 * indices ascending; off_out [batch_count][m+1] bucket offsets into the pool (row b: off[0..S'_b]);
 * sid_out [batch_count][m] the prompt sentence id of each bucket; S_out [batch_count] buckets S'_b. */
skv_status sentencekv_copy_retained(skv_ctx* ctx, int32_t layer, int32_t* keep_out, int32_t* off_out,
                                    int32_t* sid_out, int32_t* S_out, skv_stream_t stream);

/* Number of CUDA kernel launches this context has enqueued since creation. */
int64_t sentencekv_launch_count(const skv_ctx* ctx);

/* ---- kernel profiler (bench / tracing; off by default) ----
 * When on, every kernel launch of this context is bracketed by two CUDA events recorded on the
 * launching stream.  Not for use while a stream is being captured into a CUDA graph. */
typedef enum {
    SKV_K_SEGMENT = 0, /* P1 */
    SKV_K_COMPRESS = 1, /* P2 */
    SKV_K_SCORE = 2,   /* D1 */
    SKV_K_SELECT = 3,  /* D2 */
    SKV_K_ATTEND = 4,  /* D3 + D4 */
    SKV_K_RETAIN = 5,  /* NEXT-1 retention: window importance (2 tcgen05 passes), top-k, pool gather */
    SKV_K_STEP = 6,    /* D1 + D2 + D3 + D4 in one launch (decode_step, default) */
    SKV_K_OFFLOAD = 7, /* P3: the D2H copies of a layer's K and V on the ctx's copy stream (host residency) */
    SKV_K_APPEND = 8,  /* NEXT-2 decode_append: close a generated sentence into a bucket, store k / v */
    SKV_K_COUNT = 9
} skv_kernel_kind;

skv_status sentencekv_set_profiling(skv_ctx* ctx, int32_t on);

/* Tuning of sentencekv_decode_step's selection (performance only -- results are exact for any value):
 * the one-launch kernel first ranks a band of ordered-key width 2^log2 around the previous step's
 * crossing point and falls back to its general path when the crossing point left it.
 * log2 in [0, 29]; default 19.  INVALID_ARGUMENT outside the range. */
skv_status sentencekv_set_band_log2(skv_ctx* ctx, int32_t log2);

/* Synchronises, then adds the elapsed time of every profiled launch since the last read:
 * ms_out host double [SKV_K_COUNT] (total milliseconds per kind), n_out host int64 [SKV_K_COUNT]
 * (launches per kind).  Both are accumulated into (not overwritten). */
skv_status sentencekv_profile_read(skv_ctx* ctx, double* ms_out, int64_t* n_out);

#ifdef __cplusplus
}
#endif

#endif /* SENTENCEKV_H */
