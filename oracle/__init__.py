"""CPU oracle for the SentenceKV hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2504_00970_b200``) never imports it and shares no code with it.

The arithmetic lives in plain C (``oracle/skvref.c``, one function per step of the paper,
each citing its passage); this module only marshals numpy arrays into those functions and
sequences them in the order of Algorithm 1.  bf16 tensors are passed
as their raw ``uint16`` bit patterns.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "skvref.c")
_LIB = os.path.join(_HERE, "libskvref.so")

# -O2, IEEE semantics: no -ffast-math, no fp contraction (the canonical fp32 order of the
# selection arithmetic is written out explicitly, fmaf where the order says fma).
CFLAGS = ["-O2", "-fPIC", "-shared", "-std=c11", "-ffp-contract=off", "-fno-fast-math"]


def build(force: bool = False) -> str:
    """Compile ``skvref.c`` into ``libskvref.so`` (gcc).  Returns the library path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i32, i64, f32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_float
        L.skvref_segment.argtypes = [P, i32, P, i32, i32, P]
        L.skvref_segment.restype = i32
        L.skvref_embed.argtypes = [P, i32, P, i32, P]
        L.skvref_embed.restype = None
        L.skvref_qs_append_mean.argtypes = [P, P, P, i32, i32, P]
        L.skvref_qs_append_mean.restype = None
        L.skvref_qs_reset.argtypes = [P, P, i32, i32]
        L.skvref_qs_reset.restype = None
        L.skvref_group_query.argtypes = [P, i32, i32, i32, P]
        L.skvref_group_query.restype = None
        L.skvref_score.argtypes = [P, P, i32, i32, P]
        L.skvref_score.restype = None
        L.skvref_select.argtypes = [P, P, i32, i32, P, P]
        L.skvref_select.restype = i32
        L.skvref_attend.argtypes = [P, i32, P, P, i32, P, P, i32, P]
        L.skvref_attend.restype = None
        L.skvref_window_importance.argtypes = [P, P, i32, i32, i32, i32, i32, P]
        L.skvref_window_importance.restype = None
        L.skvref_retain.argtypes = [P, i32, i32, P]
        L.skvref_retain.restype = i32
        L.skvref_retained_buckets.argtypes = [P, i32, P, i32, P, P]
        L.skvref_retained_buckets.restype = i32
        L.skvref_equal_chunks.argtypes = [i32, i32, i32, P]
        L.skvref_equal_chunks.restype = i32
        L.skvref_outlier_threshold.argtypes = [P, i32, ctypes.c_double]
        L.skvref_outlier_threshold.restype = i32
        L.skvref_select_skip.argtypes = [P, P, i32, i32, P, P]
        L.skvref_select_skip.restype = i32
        L.skvref_quest_meta.argtypes = [P, i32, i32, i32, P, P]
        L.skvref_quest_meta.restype = None
        L.skvref_quest_score.argtypes = [P, i32, P, P, i32, i32, P]
        L.skvref_quest_score.restype = None
        L.skvref_kv_bytes.argtypes = [i64, i64, i64, i64, i64]
        L.skvref_kv_bytes.restype = i64
        L.skvref_f32_to_bf16.argtypes = [f32]
        L.skvref_f32_to_bf16.restype = ctypes.c_uint16
        L.skvref_bf16_to_f32.argtypes = [ctypes.c_uint16]
        L.skvref_bf16_to_f32.restype = f32
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ----------------------------------------------------------------------------- steps


def segment(tokens, boundary_ids, tau: int) -> np.ndarray:
    """P1: sentence offsets ``off[S+1]`` of one prompt (int32)."""
    tokens = _c(tokens, np.int32)
    bset = _c(boundary_ids, np.int32)
    off = np.zeros(len(tokens) + 1, dtype=np.int32)
    S = lib().skvref_segment(_p(tokens), len(tokens), _p(bset), len(bset), int(tau), _p(off))
    return off[: S + 1].copy()


def embed(K_bits, off) -> np.ndarray:
    """P2, Eq. 1: mean key per sentence of one (b, g) unit.  K_bits uint16 [L][d]."""
    K_bits = _c(K_bits, np.uint16)
    off = _c(off, np.int32)
    S = len(off) - 1
    d = K_bits.shape[1]
    E = np.zeros((S, d), dtype=np.uint16)
    lib().skvref_embed(_p(K_bits), d, _p(off), S, _p(E))
    return E


def qs_append_mean(Sq, cnt, q_bits):
    """D1, Eq. 2: Sq += q, cnt += 1, returns qbar = Sq / cnt.  In-place on Sq/cnt."""
    Hq, d = q_bits.shape
    q_bits = _c(q_bits, np.uint16)
    qbar = np.zeros((Hq, d), dtype=np.float32)
    lib().skvref_qs_append_mean(_p(Sq), _p(cnt), _p(q_bits), Hq, d, _p(qbar))
    return qbar


def qs_reset(Sq, cnt):
    """D1 reset at a sentence boundary (Alg. 1 l.19-21)."""
    lib().skvref_qs_reset(_p(Sq), _p(cnt), Sq.shape[0], Sq.shape[1])


def group_query(qbar, grp: int, g: int) -> np.ndarray:
    """GQA group query qt_g = sum of the group's mean queries (reading A9)."""
    qbar = _c(qbar, np.float32)
    qt = np.zeros(qbar.shape[1], dtype=np.float32)
    lib().skvref_group_query(_p(qbar), grp, qbar.shape[1], g, _p(qt))
    return qt


def score(qt, E_bits) -> np.ndarray:
    """D1 similarity qbar^T kbar, canonical fp32 order."""
    qt = _c(qt, np.float32)
    E_bits = _c(E_bits, np.uint16)
    S, d = E_bits.shape
    out = np.zeros(S, dtype=np.float32)
    lib().skvref_score(_p(qt), _p(E_bits), S, d, _p(out))
    return out


def select(scores, off, tau: int):
    """D2: ascending selected ids and the number of selected tokens."""
    scores = _c(scores, np.float32)
    off = _c(off, np.int32)
    S = len(off) - 1
    ids = np.zeros(max(S, 1), dtype=np.int32)
    ntok = np.zeros(1, dtype=np.int32)
    n = lib().skvref_select(_p(scores), _p(off), S, int(tau), _p(ids), _p(ntok))
    return ids[:n].copy(), int(ntok[0])


def attend(q_bits, K_bits, V_bits, off, ids) -> np.ndarray:
    """D4, Eq. 3 in fp64 over the selected sentences' tokens.  q_bits [grp][d]."""
    q_bits = _c(q_bits, np.uint16)
    K_bits = _c(K_bits, np.uint16)
    V_bits = _c(V_bits, np.uint16)
    off = _c(off, np.int32)
    ids = _c(ids, np.int32)
    grp, d = q_bits.shape
    out = np.zeros((grp, d), dtype=np.float64)
    lib().skvref_attend(_p(q_bits), grp, _p(K_bits), _p(V_bits), d, _p(off), _p(ids), len(ids), _p(out))
    return out


def full_attend(q_bits, K_bits, V_bits) -> np.ndarray:
    """O-FULL: Eq. 3 over all L tokens (the Full-KV baseline) -- one sentence [0, L)."""
    L = K_bits.shape[0]
    return attend(q_bits, K_bits, V_bits, np.array([0, L], np.int32), np.array([0], np.int32))


def window_importance(qw_bits, K_bits) -> np.ndarray:
    """NEXT-1 token importance: alpha fp64 [L-N] of one sequence from the window queries
    qw_bits [N][Hq][d] and the keys K_bits [G][L][d] (reading A21)."""
    qw_bits = _c(qw_bits, np.uint16)
    K_bits = _c(K_bits, np.uint16)
    N, Hq, d = qw_bits.shape
    G, L, _ = K_bits.shape
    assert L > N >= 1
    alpha = np.zeros(L - N, dtype=np.float64)
    lib().skvref_window_importance(_p(qw_bits), _p(K_bits), N, Hq, G, L, d, _p(alpha))
    return alpha


def retain(alpha, k: int) -> np.ndarray:
    """NEXT-1 global top-k tokens by alpha, ascending indices (int32)."""
    alpha = _c(alpha, np.float64)
    keep = np.zeros(max(1, min(int(k), len(alpha))), dtype=np.int32)
    m = lib().skvref_retain(_p(alpha), len(alpha), int(k), _p(keep))
    return keep[:m].copy()


def retained_buckets(off, keep):
    """NEXT-1 sentence buckets over the retained pool (reading A25): (off2 [S'+1], sid [S'])."""
    off = _c(off, np.int32)
    keep = _c(keep, np.int32)
    S = len(off) - 1
    off2 = np.zeros(S + 1, dtype=np.int32)
    sid = np.zeros(max(1, S), dtype=np.int32)
    S2 = lib().skvref_retained_buckets(_p(off), S, _p(keep), len(keep), _p(off2), _p(sid))
    return off2[: S2 + 1].copy(), sid[:S2].copy()


def equal_chunks(L: int, S: int, tau: int) -> np.ndarray:
    """NEXT-3 equal-size chunks (Sec. 6.1; reading A26): offsets of as many chunks as sentences."""
    off = np.zeros(L + 1, dtype=np.int32)
    n = lib().skvref_equal_chunks(int(L), int(S), int(tau), _p(off))
    return off[: n + 1].copy()


def outlier_threshold(off, n: float) -> int:
    """NEXT-3 outlier split (reading A27): T = floor(mean + n * std) of the sentence lengths."""
    off = _c(off, np.int32)
    return int(lib().skvref_outlier_threshold(_p(off), len(off) - 1, float(np.float32(n))))


def select_skip(scores, off, tau: int):
    """NEXT-3 skip-and-continue budget fill (alternative to A13): ascending ids and selected tokens."""
    scores = _c(scores, np.float32)
    off = _c(off, np.int32)
    S = len(off) - 1
    ids = np.zeros(max(S, 1), dtype=np.int32)
    ntok = np.zeros(1, dtype=np.int32)
    n = lib().skvref_select_skip(_p(scores), _p(off), S, int(tau), _p(ids), _p(ntok))
    return ids[:n].copy(), int(ntok[0])


def quest_meta(K_bits, P: int):
    """NEXT-4 Quest pages (App. Quest): per-page min / max keys, bf16 bits [np][d] each."""
    K_bits = _c(K_bits, np.uint16)
    L, d = K_bits.shape
    npg = (L + P - 1) // P
    mn = np.zeros((npg, d), dtype=np.uint16)
    mx = np.zeros((npg, d), dtype=np.uint16)
    lib().skvref_quest_meta(_p(K_bits), L, d, int(P), _p(mn), _p(mx))
    return mn, mx


def quest_score(q_bits, mn, mx) -> np.ndarray:
    """NEXT-4 Quest bound sum_h sum_j max(q_j mn_j, q_j mx_j) per page (reading A28), q_bits [grp][d]."""
    q_bits = _c(q_bits, np.uint16)
    mn = _c(mn, np.uint16)
    mx = _c(mx, np.uint16)
    grp, d = q_bits.shape
    out = np.zeros(mn.shape[0], dtype=np.float32)
    lib().skvref_quest_score(_p(q_bits), grp, _p(mn), _p(mx), mn.shape[0], d, _p(out))
    return out


def retained_count(r: float, tau: int) -> int:
    """floor(r * tau) (reading A20), the number of tokens the retention keeps."""
    import math

    return int(math.floor(float(np.float32(r)) * int(tau)))


def kv_bytes(M, H, d, tokens, elem_bytes=2) -> int:
    """App. Cost(t) written out: M*H*(L+t)*d*2*elem_bytes."""
    return int(lib().skvref_kv_bytes(M, H, d, tokens, elem_bytes))


def synth_free_bf16_to_f32(bits) -> np.ndarray:
    """bf16 bit patterns -> fp32 (exact widening)."""
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16_bits(x: float) -> int:
    return int(lib().skvref_f32_to_bf16(float(x)))


# ------------------------------------------------------------------- Algorithm 1 driver


class Oracle:
    """Algorithm 1 for the hot path, one object per prompt batch.

    Shapes follow the ABI: tokens [B][L]; per layer K, V bf16 bits [B][G][L][d];
    per decode step and layer q bf16 bits [B][Hq][d] and the input token ids [B].
    """

    BUCKETS_SENTENCE, BUCKETS_EQUAL, BUCKETS_QUEST = 0, 1, 2

    def __init__(self, tokens, boundary_ids, tau: int, layers: int, q_heads: int, kv_heads: int, d: int,
                 obs_window: int = 0, semantic_factor: float = 2.0, bucket_mode: int = 0, chunk_size: int = 0,
                 outlier_n: float = 0.0, query_mode: int = 0, fill_mode: int = 0, max_generated: int = 0):
        self.tokens = np.asarray(tokens, dtype=np.int32)
        self.B = self.tokens.shape[0]
        self.bset = np.asarray(boundary_ids, dtype=np.int32)
        self.tau = int(tau)
        self.M, self.Hq, self.G, self.d = layers, q_heads, kv_heads, d
        self.grp = q_heads // kv_heads
        # P1: segmentation, shared by all layers and heads (Alg. 1 line 2), or a NEXT-3 / NEXT-4 variant
        self.bucket_mode, self.chunk_size, self.outlier_n = bucket_mode, chunk_size, outlier_n
        self.query_mode, self.fill_mode = query_mode, fill_mode
        L = self.tokens.shape[1]
        self.off = []
        for b in range(self.B):
            off = segment(self.tokens[b], self.bset, self.tau)
            if bucket_mode == self.BUCKETS_EQUAL:
                off = equal_chunks(L, len(off) - 1, self.tau)
            elif bucket_mode == self.BUCKETS_QUEST:
                off = np.minimum(np.arange(0, L + chunk_size, chunk_size), L).astype(np.int32)
                off = np.unique(off)
            elif outlier_n > 0:
                T = outlier_threshold(off, outlier_n)
                off = segment(self.tokens[b], self.bset, min(self.tau, T))
            self.off.append(off)
        self.N, self.r = int(obs_window), float(semantic_factor)
        self.E = {}  # layer -> list[b][g] of E bits
        self.K = {}
        self.V = {}
        # NEXT-1 retention (obs_window > 0): per layer, per b: alpha, retained token ids, bucket
        # offsets over the pool and the sentence id of each bucket; K/V above are then the pools
        self.alpha, self.keep, self.loff, self.sid, self.win = {}, {}, {}, {}, {}
        # NEXT-2 local segment and growth (max_generated > 0; reading A29): per layer, per b: the
        # generated tokens' K/V, the start of the current (unfinished) generated sentence, whether the
        # sentence ended at the last appended token, and the bucket offsets extended by the completed
        # generated sentences (rows >= L are generated rows)
        self.max_gen = int(max_generated)
        self.gK, self.gV, self.ghot, self.gpend, self.goff = {}, {}, {}, {}, {}
        self.Sq = np.zeros((layers, self.B, q_heads, d), dtype=np.float32)
        self.cnt = np.zeros((layers, self.B), dtype=np.int32)

    def offsets(self, layer: int, b: int) -> np.ndarray:
        """Bucket offsets the decode of (layer, b) ranks: the prompt's sentences, the retained buckets,
        or (NEXT-2) the prompt's sentences followed by the completed generated sentences."""
        if layer in self.goff:
            return self.goff[layer][b]
        return self.loff[layer][b] if layer in self.loff else self.off[b]

    def decode_append(self, layer: int, k_bits, v_bits, input_token):
        """NEXT-2 (P:456 'append ... and repeat'; reading A29), before the step's ranking: a sentence of
        generated text that ended at the previous step becomes a retrievable bucket (Eq. 1 mean of its
        keys appended to the layer's embeddings); then this step's token K/V (k_bits, v_bits bf16 bits
        [B][G][d]) joins the local segment, and if the token is a boundary its sentence ends here."""
        L = self.tokens.shape[1]
        if layer not in self.gK:
            self.gK[layer] = [np.zeros((self.G, 0, self.d), np.uint16) for _ in range(self.B)]
            self.gV[layer] = [np.zeros((self.G, 0, self.d), np.uint16) for _ in range(self.B)]
            self.ghot[layer] = [0] * self.B
            self.gpend[layer] = [False] * self.B
            self.goff[layer] = [self.offsets(layer, b).copy() for b in range(self.B)]
            if layer in self.loff:  # retention: bucket ids -> sentence ids, extended by the generated ones
                self.gsid0 = getattr(self, "gsid0", {})
                self.gsid0[layer] = [len(self.sid[layer][b]) for b in range(self.B)]
                # the observation window's rows are the local segment when decoding starts (A29): the
                # store begins with them, and they close with the first generated sentence
                self.gK[layer] = [self.win[layer][b][0].copy() for b in range(self.B)]
                self.gV[layer] = [self.win[layer][b][1].copy() for b in range(self.B)]
        # store row i (generated token i, or with retention the window's rows first) is row L + i, or
        # (retention) m + i behind the retained pool
        base = [(L if layer not in self.loff else self.loff[layer][b][-1]) for b in range(self.B)]
        for b in range(self.B):
            n = self.gK[layer][b].shape[1]
            if self.gpend[layer][b]:
                h = self.ghot[layer][b]
                for g in range(self.G):
                    e = embed(self.gK[layer][b][g, h:n], np.array([0, n - h], np.int32))
                    self.E[layer][b][g] = np.concatenate([self.E[layer][b][g], e])
                self.goff[layer][b] = np.append(self.goff[layer][b], np.int32(base[b] + n))
                if layer in self.loff:  # generated sentence k of sequence b is sentence S_b + k
                    k = len(self.goff[layer][b]) - 2 - self.gsid0[layer][b]
                    self.sid[layer][b] = np.append(self.sid[layer][b], np.int32(len(self.off[b]) - 1 + k))
                self.ghot[layer][b] = n
                self.gpend[layer][b] = False
            self.gK[layer][b] = np.concatenate([self.gK[layer][b], k_bits[b][:, None, :]], axis=1)
            self.gV[layer][b] = np.concatenate([self.gV[layer][b], v_bits[b][:, None, :]], axis=1)
            # the sentence ends at a boundary token (A11) or when it reaches tau tokens (the A5 cap)
            if int(input_token[b]) in set(self.bset.tolist()) or n + 1 - self.ghot[layer][b] >= self.tau:
                self.gpend[layer][b] = True

    def prefill_layer(self, layer: int, K_bits, V_bits, q_window=None):
        """Alg. 1 lines 3-8 for one layer: Eq. 1 mean keys.  Without a window (reading A6) every
        token of a sentence is kept (A19); with one (NEXT-1, q_window bf16 bits [B][N][Hq][d]):
        alpha (line 4), global top-floor(r*tau) retention (line 5), Eq. 1 over the retained tokens
        of each sentence (line 6), and the retained pool kept for retrieval (line 7)."""
        if q_window is None:
            self.K[layer], self.V[layer] = K_bits, V_bits
            if self.bucket_mode == self.BUCKETS_QUEST:  # page bounds instead of Eq. 1 means
                self.E[layer] = [[quest_meta(K_bits[b, g], self.chunk_size) for g in range(self.G)] for b in range(self.B)]
            else:
                self.E[layer] = [[embed(K_bits[b, g], self.off[b]) for g in range(self.G)] for b in range(self.B)]
            return
        k = retained_count(self.r, self.tau)
        al, kp, lo, sd, Kp, Vp = [], [], [], [], [], []
        for b in range(self.B):
            a = window_importance(q_window[b], K_bits[b])
            keep = retain(a, k)
            off2, sid = retained_buckets(self.off[b], keep)
            al.append(a)
            kp.append(keep)
            lo.append(off2)
            sd.append(sid)
            Kp.append(np.ascontiguousarray(K_bits[b][:, keep]))
            Vp.append(np.ascontiguousarray(V_bits[b][:, keep]))
        self.alpha[layer], self.keep[layer], self.loff[layer], self.sid[layer] = al, kp, lo, sd
        # the observation window itself (positions >= L - N): not a candidate, attended every step (A25)
        L = K_bits.shape[2]
        self.win[layer] = [(np.ascontiguousarray(K_bits[b][:, L - self.N:]), np.ascontiguousarray(V_bits[b][:, L - self.N:]))
                           for b in range(self.B)]
        self.K[layer], self.V[layer] = Kp, Vp  # [b] -> [G][m][d]
        self.E[layer] = [[embed(Kp[b][g], lo[b]) for g in range(self.G)] for b in range(self.B)]

    def decode_select(self, layer: int, q_bits, input_token):
        """Alg. 1 lines 14-17: append q_t, qbar (Eq. 2), similarity, budgeted retrieval.

        Returns (scores[b][g], ids[b][g], ntok[b][g]); applies the boundary reset (A11)
        after the step."""
        scores, ids, ntok = [], [], []
        for b in range(self.B):
            Sq = self.Sq[layer, b]
            cnt = self.cnt[layer, b : b + 1]
            qbar = qs_append_mean(Sq, cnt, q_bits[b])
            if self.query_mode == 1:  # NEXT-3 current-token query (Sec. 6.2)
                qbar = synth_free_bf16_to_f32(q_bits[b])
            sb, ib, nb = [], [], []
            for g in range(self.G):
                if self.bucket_mode == self.BUCKETS_QUEST:  # Quest ranks by the current query's bound
                    mn, mx = self.E[layer][b][g]
                    sc = quest_score(q_bits[b, g * self.grp:(g + 1) * self.grp], mn, mx)
                else:
                    qt = group_query(qbar, self.grp, g)
                    sc = score(qt, self.E[layer][b][g])
                fn = select_skip if self.fill_mode == 1 else select
                sel, n = fn(sc, self.offsets(layer, b), self.tau)
                sb.append(sc)
                ib.append(sel)
                nb.append(n)
            scores.append(sb)
            ids.append(ib)
            ntok.append(nb)
            if int(input_token[b]) in set(self.bset.tolist()):
                qs_reset(Sq, cnt)
        return scores, ids, ntok

    def decode_attend(self, layer: int, q_bits, ids):
        """Alg. 1 line 19 / Eq. 3 over the selection of this layer: O fp64 [B][Hq][d].  NEXT-2: the
        selected buckets (prompt rows, then generated rows) plus the local segment -- the tokens of the
        unfinished generated sentence, attended uncharged (reading A29).  NEXT-1: the selected buckets
        of the retained pool plus the observation window (reading A25)."""
        O = np.zeros((self.B, self.Hq, self.d), dtype=np.float64)
        for b in range(self.B):
            for g in range(self.G):
                h0 = g * self.grp
                # the attended rows, written out: selected buckets, the observation window (retention),
                # the sentence being generated (NEXT-2); rows index the concatenation of the context (or
                # the retained pool), the window and the generated tokens
                K, V = self.K[layer][b][g], self.V[layer][b][g]
                off = self.offsets(layer, b)
                rows = [np.arange(off[s], off[s + 1]) for s in ids[b][g]]
                if layer in self.win and layer not in self.gK:  # (with NEXT-2 the window is in the store)
                    wk, wv = self.win[layer][b]
                    rows.append(np.arange(K.shape[0], K.shape[0] + self.N))
                    K = np.concatenate([K, wk[g]])
                    V = np.concatenate([V, wv[g]])
                if layer in self.gK:
                    n, h = self.gK[layer][b].shape[1], self.ghot[layer][b]
                    rows.append(np.arange(K.shape[0] + h, K.shape[0] + n))
                    K = np.concatenate([K, self.gK[layer][b][g]])
                    V = np.concatenate([V, self.gV[layer][b][g]])
                idx = np.concatenate(rows).astype(np.int64) if rows else np.zeros(0, np.int64)
                Ka, Va = np.ascontiguousarray(K[idx]), np.ascontiguousarray(V[idx])
                O[b, h0 : h0 + self.grp] = attend(q_bits[b, h0 : h0 + self.grp], Ka, Va,
                                                  np.array([0, len(idx)], np.int32), np.array([0], np.int32))
        return O
