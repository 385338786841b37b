/*
 * skvref.c -- plain, slow, obviously-correct CPU oracle for the SentenceKV hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2504_00970_b200/) never links, imports or calls it, and shares no code,
 * header, table or constant generator with it.
 *
 * Paper: "SentenceKV" (arXiv 2504.00970), /root/reference/PAPER.md.  Citations are
 * "P:<line>" = PAPER.md line, with the section / equation / algorithm they fall in.
 * Readings of points the paper leaves open are numbered A1..A22 and listed in
 * DESIGN.md section "Readings"; each function names the ones it depends on.
 *
 * Numeric regimes (DESIGN.md "Readings" A7, A23):
 *   - Selection-deciding arithmetic (sentence mean keys, mean query, scores) is written
 *     in IEEE fp32 in one fixed order (the "canonical order" spelled out per function),
 *     because a floating-point value decides an integer result (the selected sentence
 *     ids) and the task requires both sides to take that decision in the same precision.
 *   - Attention (Eq. 3) is evaluated in fp64.
 * Build: gcc -O2 -fPIC -shared -ffp-contract=off (no -ffast-math), see oracle/build.sh.
 *
 * Parity status per function: every function below is pinned by tests/test_oracle_*.py
 * (worked examples, closed forms, brute force, library routines); none is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- bf16 helpers */

/* bf16 -> fp32 is exact: the bf16 bit pattern is the upper half of the fp32 one. */
static float bf16_to_f32(uint16_t h) {
    uint32_t u = ((uint32_t)h) << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

/* fp32 -> bf16, round to nearest, ties to even (reading A7).  NaN stays a quiet NaN. */
static uint16_t f32_to_bf16_rne(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x0040u);
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    return (uint16_t)(u >> 16);
}

uint16_t skvref_f32_to_bf16(float f) { return f32_to_bf16_rne(f); }
float skvref_bf16_to_f32(uint16_t h) { return bf16_to_f32(h); }

/* ------------------------------------------------------------ P1: segmentation */

static int is_boundary(int32_t tok, const int32_t* bset, int32_t nb) {
    for (int32_t i = 0; i < nb; ++i)
        if (bset[i] == tok) return 1;
    return 0;
}

/*
 * Split a prompt into sentence buckets "according to punctuation" (Sec. 4.1;
 * Alg. 1 line 2; boundary examples "period, question mark" P:430, Sec. 4.2).
 * Readings: A1 boundary = membership in a caller-given token-id set; A2 the boundary
 * token ends (belongs to) its sentence; A3 consecutive boundaries are not merged;
 * A4 tokens after the last boundary form the last sentence; A5 a run that reaches tau
 * tokens is closed there (tau-cap), so no sentence is longer than the budget.
 *
 * Output: off[0..S] with off[0] = 0, off[S] = L; sentence s = tokens [off[s], off[s+1]).
 * off must have room for L+1 entries.  Returns S.
 */
int32_t skvref_segment(const int32_t* tokens, int32_t L, const int32_t* bset, int32_t nb,
                       int32_t tau, int32_t* off) {
    int32_t S = 0, cur_len = 0;
    off[0] = 0;
    for (int32_t i = 0; i < L; ++i) {
        cur_len += 1;
        if (is_boundary(tokens[i], bset, nb) || i == L - 1 || cur_len == tau) {
            S += 1;
            off[S] = i + 1; /* close sentence [off[S-1], i+1) */
            cur_len = 0;
        }
    }
    return S;
}

/* ------------------------------------------------------- P2: Eq. 1 mean keys */

/*
 * Sentence semantic vector, Eq. 1 (Sec. 4.1):  kbar_{s,h} = (1/|S_s|) sum_{x in S_s} k_{x,h}
 * for one (sequence, KV head) unit.  Reading A6: S_s = all member tokens of sentence s
 * (full K/V kept, north_star); A7: fp32 sum, canonical order = ascending token index,
 * one IEEE division by n, then bf16 round-to-nearest-even.
 *
 * K: bf16 bits [L][d] (row t = key of token t for this head); off: [S+1]; E: bf16 bits [S][d].
 */
void skvref_embed(const uint16_t* K, int32_t d, const int32_t* off, int32_t S, uint16_t* E) {
    for (int32_t s = 0; s < S; ++s) {
        int32_t a = off[s], b = off[s + 1];
        float n = (float)(b - a);
        for (int32_t j = 0; j < d; ++j) {
            float acc = 0.0f;
            for (int32_t t = a; t < b; ++t) acc = acc + bf16_to_f32(K[(int64_t)t * d + j]);
            float mean = acc / n;
            E[(int64_t)s * d + j] = f32_to_bf16_rne(mean);
        }
    }
}

/* -------------------------------------------------- D1: Eq. 2 sentence query cache */

/*
 * Sentence query cache Q_s and mean query, Eq. 2 (Sec. 4.2; Alg. 1 lines 13-15,
 * P:586-588):  append q_t to Q_s, qbar = (1/|Q_s|) sum_{t in Q_s} q_t.
 * Q_s is represented by its running fp32 sum Sq[Hq][d] and count *cnt (A10: qbar includes
 * the current q_t; canonical order = steps in time order, one fp32 add per step, then one
 * IEEE division).  The reset at a sentence boundary (Alg. 1 lines 19-21) is applied
 * by skvref_qs_reset after the step (A11).
 *
 * q: bf16 bits [Hq][d] of the current token; qbar: fp32 [Hq][d] out.
 */
void skvref_qs_append_mean(float* Sq, int32_t* cnt, const uint16_t* q, int32_t Hq, int32_t d,
                           float* qbar) {
    *cnt += 1;
    float c = (float)(*cnt);
    for (int32_t i = 0; i < Hq * d; ++i) {
        Sq[i] = Sq[i] + bf16_to_f32(q[i]);
        qbar[i] = Sq[i] / c;
    }
}

void skvref_qs_reset(float* Sq, int32_t* cnt, int32_t Hq, int32_t d) {
    for (int32_t i = 0; i < Hq * d; ++i) Sq[i] = 0.0f;
    *cnt = 0;
}

/*
 * GQA group query (reading A9): the KV head g is shared by query heads g*grp .. g*grp+grp-1;
 * the per-head similarities qbar_h^T kbar_{s,g} are ranked per KV head through
 * qt_g = sum_h qbar_h, summed in ascending h.  qbar: [Hq][d]; qt: [d].
 */
void skvref_group_query(const float* qbar, int32_t grp, int32_t d, int32_t g, float* qt) {
    for (int32_t j = 0; j < d; ++j) {
        float acc = qbar[(int64_t)(g * grp) * d + j];
        for (int32_t h = 1; h < grp; ++h) acc = acc + qbar[(int64_t)(g * grp + h) * d + j];
        qt[j] = acc;
    }
}

/* ------------------------------------------------------------ D1: similarity score */

/*
 * Similarity S(qbar, kbar_s) = qbar^T kbar_s (Sec. 4.2; Alg. 1 line 16),
 * for every sentence s of one unit.  Canonical fp32 order (reading A23): split d into d/8
 * lanes; lane l computes p_l = qt[8l]*e[8l], then p_l = fma(qt[8l+i], e[8l+i], p_l) for
 * i = 1..7; then for w = d/16, d/32, ..., 1: p_l = p_l + p_{l+w} for l < w; score = p_0.
 * qt: fp32 [d]; E: bf16 bits [S][d]; score: fp32 [S].  d must be a multiple of 16.
 */
void skvref_score(const float* qt, const uint16_t* E, int32_t S, int32_t d, float* score) {
    float p[64];
    int32_t lanes = d / 8;
    for (int32_t s = 0; s < S; ++s) {
        const uint16_t* e = E + (int64_t)s * d;
        for (int32_t l = 0; l < lanes; ++l) {
            float acc = qt[8 * l] * bf16_to_f32(e[8 * l]);
            for (int32_t i = 1; i < 8; ++i) acc = fmaf(qt[8 * l + i], bf16_to_f32(e[8 * l + i]), acc);
            p[l] = acc;
        }
        for (int32_t w = lanes / 2; w >= 1; w /= 2)
            for (int32_t l = 0; l < w; ++l) p[l] = p[l] + p[l + w];
        score[s] = p[0];
    }
}

/* ------------------------------------------------------- D2: budgeted selection */

/* Order-preserving map of an fp32 score to u32 (reading A14): -0 == +0, NaN ranks last. */
static uint32_t ordered_u32(float x) {
    if (x != x) return 0u;
    if (x == 0.0f) x = 0.0f;
    uint32_t u;
    memcpy(&u, &x, 4);
    return (u >> 31) ? ~u : (u | 0x80000000u);
}

static int cmp_key_desc(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return (x < y) ? 1 : (x > y) ? -1 : 0;
}

static int cmp_i32_asc(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

/*
 * Ranked retrieval under the budget (Sec. 4.2: "rank all sentence buckets by their
 * similarity scores and retrieve tokens from the most relevant buckets in descending order
 * ... until we reach our token budget tau"; Alg. 1 line 17).
 * Readings: A13 whole sentences only, the maximal prefix of the ranking whose lengths sum to
 * <= tau (stop at the first sentence that does not fit); A14 ties -> lowest sentence index
 * first, -0 == +0, NaN last; A15 tau applies per (sequence, layer, KV head).
 *
 * score: [S]; off: [S+1] sentence offsets; ids: out, ascending selected sentence ids
 * (room for S); *ntok: out, number of selected tokens.  Returns the number of sentences.
 */
int32_t skvref_select(const float* score, const int32_t* off, int32_t S, int32_t tau, int32_t* ids,
                      int32_t* ntok) {
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(S > 0 ? S : 1));
    for (int32_t s = 0; s < S; ++s)
        keys[s] = ((uint64_t)ordered_u32(score[s]) << 32) | (uint64_t)(0xffffffffu - (uint32_t)s);
    qsort(keys, (size_t)S, sizeof(uint64_t), cmp_key_desc);
    int32_t count = 0, tot = 0;
    for (int32_t r = 0; r < S; ++r) {
        int32_t s = (int32_t)(0xffffffffu - (uint32_t)(keys[r] & 0xffffffffu));
        int32_t n = off[s + 1] - off[s];
        if (tot + n > tau) break;
        tot += n;
        ids[count++] = s;
    }
    qsort(ids, (size_t)count, sizeof(int32_t), cmp_i32_asc);
    free(keys);
    *ntok = tot;
    return count;
}

/* -------------------------------------------------- D4: Eq. 3 restricted attention */

/*
 * Attention over the retrieved tokens only, Eq. 3 (Sec. 4.2; Alg. 1 line 19,
 * P:592):  O = softmax(q K_tau^T / sqrt(d)) V_tau, in fp64 (A16: current token's query q_t,
 * scale 1/sqrt(d), no mask; A17: the retrieved context tokens only).
 * The attended set is the union of the selected sentences' token ranges (O-GATHER), read
 * from the original K/V.
 *
 * q: bf16 bits [grp][d] (the query heads of this KV head); K, V: bf16 bits [L][d];
 * off: [S+1]; ids: [nsel] selected sentences; out: fp64 [grp][d].
 */
void skvref_attend(const uint16_t* q, int32_t grp, const uint16_t* K, const uint16_t* V, int32_t d,
                   const int32_t* off, const int32_t* ids, int32_t nsel, double* out) {
    int32_t n = 0;
    for (int32_t i = 0; i < nsel; ++i) n += off[ids[i] + 1] - off[ids[i]];
    int32_t* tok = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    double* z = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    int32_t m = 0;
    for (int32_t i = 0; i < nsel; ++i)
        for (int32_t t = off[ids[i]]; t < off[ids[i] + 1]; ++t) tok[m++] = t;
    double scale = 1.0 / sqrt((double)d);
    for (int32_t h = 0; h < grp; ++h) {
        double zmax = -INFINITY;
        for (int32_t i = 0; i < n; ++i) {
            double acc = 0.0;
            for (int32_t j = 0; j < d; ++j)
                acc += (double)bf16_to_f32(q[(int64_t)h * d + j]) *
                       (double)bf16_to_f32(K[(int64_t)tok[i] * d + j]);
            z[i] = acc * scale;
            if (z[i] > zmax) zmax = z[i];
        }
        double denom = 0.0;
        for (int32_t i = 0; i < n; ++i) {
            z[i] = exp(z[i] - zmax);
            denom += z[i];
        }
        for (int32_t j = 0; j < d; ++j) {
            double acc = 0.0;
            for (int32_t i = 0; i < n; ++i) acc += z[i] * (double)bf16_to_f32(V[(int64_t)tok[i] * d + j]);
            out[(int64_t)h * d + j] = acc / denom;
        }
    }
    free(tok);
    free(z);
}

/* ------------------------------- NEXT-1: importance-filtered retention (Sec. 4.1) */

/*
 * Token importance, Sec. 4.1 "Token importance measurement" (Alg. 1 line 4):
 * the last N prompt tokens are the observation window; every window token attends to the
 * tokens before it and "for each token i in the preceding positions, we calculate its
 * importance score alpha_i by summing the attention scores it receives from all tokens in the
 * observation window, across all the attention heads".
 * Reading A21: window token w sits at position p = L-N+w and its attention is the softmax of
 * q_w . k_j / sqrt(d) over its causal prefix j = 0..p (the window tokens before it included,
 * as in a forward pass); alpha_j sums those probabilities over every window token and every
 * query head h (KV head h / grp under GQA, reading A9) for the candidates j in [0, L-N).
 * Evaluated in fp64.
 *
 * qw: bf16 bits [N][Hq][d] (window queries); K: bf16 bits [G][L][d] (keys of one sequence,
 * all KV heads); alpha: fp64 out [L-N].  Requires L > N >= 1.
 */
void skvref_window_importance(const uint16_t* qw, const uint16_t* K, int32_t N, int32_t Hq, int32_t G,
                              int32_t L, int32_t d, double* alpha) {
    const int32_t grp = Hq / G, n_cand = L - N;
    double* z = (double*)malloc(sizeof(double) * (size_t)L);
    double scale = 1.0 / sqrt((double)d);
    for (int32_t j = 0; j < n_cand; ++j) alpha[j] = 0.0;
    for (int32_t w = 0; w < N; ++w) {
        int32_t p = L - N + w; /* position of the window token; it sees keys 0..p */
        for (int32_t h = 0; h < Hq; ++h) {
            const uint16_t* q = qw + ((int64_t)w * Hq + h) * d;
            const uint16_t* Kg = K + (int64_t)(h / grp) * L * d;
            double zmax = -INFINITY;
            for (int32_t j = 0; j <= p; ++j) {
                double acc = 0.0;
                for (int32_t c = 0; c < d; ++c)
                    acc += (double)bf16_to_f32(q[c]) * (double)bf16_to_f32(Kg[(int64_t)j * d + c]);
                z[j] = acc * scale;
                if (z[j] > zmax) zmax = z[j];
            }
            double denom = 0.0;
            for (int32_t j = 0; j <= p; ++j) {
                z[j] = exp(z[j] - zmax);
                denom += z[j];
            }
            for (int32_t j = 0; j < n_cand; ++j) alpha[j] += z[j] / denom;
        }
    }
    free(z);
}

typedef struct {
    double a;
    int32_t i;
} skvref_alpha_idx;

static int cmp_alpha_desc(const void* x, const void* y) {
    const skvref_alpha_idx* a = (const skvref_alpha_idx*)x;
    const skvref_alpha_idx* b = (const skvref_alpha_idx*)y;
    if (a->a > b->a) return -1;
    if (a->a < b->a) return 1;
    return (a->i > b->i) - (a->i < b->i); /* ties: lowest token index first */
}

/*
 * Token selection, Sec. 4.1 "Token selection within sentence buckets": "we select
 * the top floor(r*tau) tokens with the highest alpha_i values across all sentence buckets"
 * (global, App. "Effect of Sentence Length"; Alg. 1 line 5).  Readings: A20
 * k = floor(r*tau) is computed by the caller; A21 ties -> lowest token index first.
 *
 * alpha: [n] (fp64 here; the GPU decides in fp32, reading A24); keep: out, the
 * retained token indices in ascending order (room for min(k, n)).  Returns min(k, n).
 */
int32_t skvref_retain(const double* alpha, int32_t n, int32_t k, int32_t* keep) {
    int32_t m = k < n ? k : n;
    if (m <= 0) return 0;
    skvref_alpha_idx* v = (skvref_alpha_idx*)malloc(sizeof(skvref_alpha_idx) * (size_t)n);
    for (int32_t i = 0; i < n; ++i) {
        v[i].a = alpha[i];
        v[i].i = i;
    }
    qsort(v, (size_t)n, sizeof(skvref_alpha_idx), cmp_alpha_desc);
    for (int32_t i = 0; i < m; ++i) keep[i] = v[i].i;
    qsort(keep, (size_t)m, sizeof(int32_t), cmp_i32_asc);
    free(v);
    return m;
}

/*
 * Sentence buckets after retention ("S_s contains the indices of retained tokens in
 * sentence s"; the retained tokens and their K/V are kept, the rest discarded).  The
 * retained tokens form a pool in token order; sentence s owns the pool range of its retained
 * tokens.  Reading A25: a sentence with no retained token has nothing to embed or retrieve and
 * is dropped from the ranking.
 *
 * off: [S+1] sentence offsets of the prompt; keep: [m] ascending retained token indices;
 * off2: out [S'+1] pool offsets of the surviving sentences; sid: out [S'] their sentence ids
 * (room for S).  Returns S'.
 */
int32_t skvref_retained_buckets(const int32_t* off, int32_t S, const int32_t* keep, int32_t m, int32_t* off2,
                                int32_t* sid) {
    int32_t S2 = 0, pos = 0;
    off2[0] = 0;
    for (int32_t s = 0; s < S; ++s) {
        int32_t c = 0;
        while (pos < m && keep[pos] < off[s + 1]) {
            if (keep[pos] >= off[s]) c += 1;
            pos += 1;
        }
        if (c > 0) {
            sid[S2] = s;
            off2[S2 + 1] = off2[S2] + c;
            S2 += 1;
        }
    }
    return S2;
}

/* ---------------------------------------- NEXT-3: paper variants on the same path */

/*
 * Equal-size chunking, Sec. 6.1 "Sentence chunking": "perform equal-sized chunking based on
 * the total number of sentences, dividing the text uniformly".  Reading A26: as many chunks as the
 * prompt has sentences, each of len = min(tau, ceil(L / S)) tokens (the last one shorter).
 * off: out [L+1]; returns the number of chunks.
 */
int32_t skvref_equal_chunks(int32_t L, int32_t S, int32_t tau, int32_t* off) {
    int32_t len = (L + S - 1) / S;
    if (len > tau) len = tau;
    if (len < 1) len = 1;
    int32_t n = 0;
    off[0] = 0;
    for (int32_t a = 0; a < L; a += len) {
        n += 1;
        off[n] = (a + len < L) ? a + len : L;
    }
    return n;
}

/*
 * Outlier split, App. "Effect of Sentence Length": "compute the mean and standard deviation
 * of sentence lengths in the input, and if a sentence exceeds mean + n x std, split it into smaller
 * sub-spans".  Reading A27: population statistics over the prompt's S sentences; the threshold is
 * T = floor(mean + n * std), evaluated as floor((L + n * sqrt(S * sum(len^2) - L^2)) / S) in IEEE
 * fp64 from exact integer sums (the same value as mean + n*std, in one written order); sentences
 * longer than T are cut into pieces of T tokens (the last piece shorter) -- segmentation with a cap
 * of min(tau, T).  Returns T (>= 1).
 */
int32_t skvref_outlier_threshold(const int32_t* off, int32_t S, double n) {
    int64_t L = off[S] - off[0], sq = 0;
    for (int32_t s = 0; s < S; ++s) {
        int64_t len = off[s + 1] - off[s];
        sq += len * len;
    }
    double var_s2 = (double)(S * sq - L * L); /* S^2 * variance, exact in int64 for these sizes */
    double t = floor(((double)L + n * sqrt(var_s2)) / (double)S);
    if (t < 1.0) t = 1.0;
    if (t > 2147483647.0) t = 2147483647.0;
    return (int32_t)t;
}

/*
 * Skip-and-continue budget fill (reading A13's alternative to the maximal prefix
 * of P:444): walk the ranking (score desc, index asc, A14); take every sentence that still fits the
 * remaining budget, skip the ones that do not, continue to the end.  Outputs as skvref_select.
 */
int32_t skvref_select_skip(const float* score, const int32_t* off, int32_t S, int32_t tau, int32_t* ids,
                           int32_t* ntok) {
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(S > 0 ? S : 1));
    for (int32_t s = 0; s < S; ++s)
        keys[s] = ((uint64_t)ordered_u32(score[s]) << 32) | (uint64_t)(0xffffffffu - (uint32_t)s);
    qsort(keys, (size_t)S, sizeof(uint64_t), cmp_key_desc);
    int32_t count = 0, tot = 0;
    for (int32_t r = 0; r < S; ++r) {
        int32_t s = (int32_t)(0xffffffffu - (uint32_t)(keys[r] & 0xffffffffu));
        int32_t n = off[s + 1] - off[s];
        if (tot + n > tau) continue;
        tot += n;
        ids[count++] = s;
    }
    qsort(ids, (size_t)count, sizeof(int32_t), cmp_i32_asc);
    free(keys);
    *ntok = tot;
    return count;
}

/* --------------------------------------- NEXT-4: Quest fixed pages (App. Quest) */

/*
 * Quest page metadata (the comparison system of App. "Quest Sensitivity to Chunk Size", P:653-660:
 * "divides the context into fixed-length chunks"; per-dimension min/max keys as in Quest,
 * SURVEY 8(f) NEXT-4): page p = tokens [p*P, min(L, (p+1)*P)); mn/mx[p][j] = min/max over the page's
 * keys of dimension j (exact: bf16 in, bf16 out).  K: bf16 bits [L][d]; mn, mx: bf16 bits [npages][d].
 */
void skvref_quest_meta(const uint16_t* K, int32_t L, int32_t d, int32_t P, uint16_t* mn, uint16_t* mx) {
    int32_t np = (L + P - 1) / P;
    for (int32_t p = 0; p < np; ++p) {
        int32_t a = p * P, b = (a + P < L) ? a + P : L;
        for (int32_t j = 0; j < d; ++j) {
            uint16_t lo = K[(int64_t)a * d + j], hi = lo;
            for (int32_t t = a + 1; t < b; ++t) {
                uint16_t v = K[(int64_t)t * d + j];
                if (bf16_to_f32(v) < bf16_to_f32(lo)) lo = v;
                if (bf16_to_f32(v) > bf16_to_f32(hi)) hi = v;
            }
            mn[(int64_t)p * d + j] = lo;
            mx[(int64_t)p * d + j] = hi;
        }
    }
}

/*
 * Quest criticality bound of every page for the query heads of one KV head (SPEC quest_rank_pages:
 * "page score = sum_h sum_dim max(q.min_key, q.max_key) per coordinate"), with the current token's
 * query (Quest ranks by q_t).  Canonical fp32 order (reading A28): t_j = max(q_j * mn_j, q_j * mx_j)
 * (IEEE products); per head: d/8 lanes, lane l: p = t[8l], then p = p + t[8l+i] for i = 1..7; then
 * for w = d/16, ..., 1: p_l = p_l + p_{l+w}; u_h = p_0; the heads summed in ascending h.
 * q: bf16 bits [grp][d]; mn, mx: bf16 bits [np][d]; score: fp32 [np].
 */
void skvref_quest_score(const uint16_t* q, int32_t grp, const uint16_t* mn, const uint16_t* mx, int32_t np,
                        int32_t d, float* score) {
    float p[64];
    int32_t lanes = d / 8;
    for (int32_t s = 0; s < np; ++s) {
        float U = 0.0f;
        for (int32_t h = 0; h < grp; ++h) {
            for (int32_t l = 0; l < lanes; ++l) {
                float acc = 0.0f;
                for (int32_t i = 0; i < 8; ++i) {
                    int32_t j = 8 * l + i;
                    float qj = bf16_to_f32(q[(int64_t)h * d + j]);
                    float a = qj * bf16_to_f32(mn[(int64_t)s * d + j]);
                    float b = qj * bf16_to_f32(mx[(int64_t)s * d + j]);
                    float t = a > b ? a : b;
                    acc = (i == 0) ? t : acc + t;
                }
                p[l] = acc;
            }
            for (int32_t w = lanes / 2; w >= 1; w /= 2)
                for (int32_t l = 0; l < w; ++l) p[l] = p[l] + p[l + w];
            U = (h == 0) ? p[0] : U + p[0];
        }
        score[s] = U;
    }
}

/* ------------------------------------------------------------ accounting */

/*
 * KV-cache bytes, App. "Memory Usage Calculation": Cost(t) = O(M x H x (L+t) x d);
 * written out as M * H * (L+t) * d * 2 (keys and values) * element bytes.
 */
int64_t skvref_kv_bytes(int64_t M, int64_t H, int64_t d, int64_t tokens, int64_t elem_bytes) {
    return M * H * tokens * d * 2 * elem_bytes;
}
