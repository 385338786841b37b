"""Seeded synthetic inputs for the SentenceKV hot path (shared by tests, bench and oracle callers).

This module holds NO arithmetic of the method: it only draws token streams, keys, values and
queries with the shapes and structure of the paper's workloads (recipe: DESIGN.md "Input
recipe").  Both the CUDA path and the CPU oracle consume the same
bytes it produces.

- Sentence lengths: clamp(round(exp(N(ln m, 0.5^2))), 2, 256); median m = 25 ("median length
  25-30"; long sentences rare), m = 20 for the tiny config.
  Each sentence = (len-1) ordinary ids + 1 id from the boundary set; the stream is cut at L.
- K/V: each sentence draws one of T = 64 topics; K_t = bf16(c[layer, g, topic] + N(0, 1)),
  V_t = bf16(N(0, 1)); c ~ N(0, I_d).  (Topic structure as in SPEC.md S:58.)
- Queries: q_t = bf16(c[layer, g(h), target] + N(0, 1)); the target topic changes whenever
  the step's input token is a boundary: generated sentences follow the prompt's length
  distribution (median 25), staggered across sequences.
"""
from __future__ import annotations

import numpy as np

# Llama-3-style punctuation ids are tokenizer-specific; any fixed set works (it is an ABI
# input).  Six ids, as SURVEY 8(d) M1 suggests.
BOUNDARY_IDS = np.array([13, 30, 0, 627, 5380, 4999], dtype=np.int32)
VOCAB_LO, VOCAB_HI = 256, 128000
N_TOPICS = 64


def _rng(*key: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(k) & 0xFFFFFFFF for k in key])))


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 bit patterns (nearest-even) -- input quantisation only."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def bf16_bits_to_f32(h: np.ndarray) -> np.ndarray:
    return (np.asarray(h, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def sentence_lengths(seed: int, b: int, L: int, median: float = 25.0, max_len: int = 256) -> np.ndarray:
    """Lengths of consecutive sentences covering at least L tokens."""
    rng = _rng(seed, 0x5E47, b)
    out, tot = [], 0
    while tot < L:
        n = np.clip(np.rint(np.exp(rng.normal(np.log(median), 0.5, size=4096))), 2, max_len).astype(np.int64)
        out.append(n)
        tot += int(n.sum())
    lens = np.concatenate(out)
    k = int(np.searchsorted(np.cumsum(lens), L)) + 1
    return lens[:k]


def token_stream(seed: int, b: int, L: int, median: float = 25.0, boundary_ids=BOUNDARY_IDS):
    """One prompt: (tokens int32 [L], topic-of-token int32 [L])."""
    lens = sentence_lengths(seed, b, L, median)
    rng = _rng(seed, 0x70C5, b)
    bset = np.asarray(boundary_ids, dtype=np.int64)
    ids = rng.integers(VOCAB_LO, VOCAB_HI, size=int(lens.sum()))
    # ordinary ids must not collide with the boundary set
    clash = np.isin(ids, bset)
    while clash.any():
        ids[clash] = rng.integers(VOCAB_LO, VOCAB_HI, size=int(clash.sum()))
        clash = np.isin(ids, bset)
    ends = np.cumsum(lens) - 1
    ids[ends] = bset[rng.integers(0, len(bset), size=len(lens))]
    topics = np.repeat(rng.integers(0, N_TOPICS, size=len(lens)), lens)
    return ids[:L].astype(np.int32), topics[:L].astype(np.int32)


def prompts(seed: int, B: int, L: int, median: float = 25.0, boundary_ids=BOUNDARY_IDS):
    toks, tops = zip(*(token_stream(seed, b, L, median, boundary_ids) for b in range(B)))
    return np.stack(toks), np.stack(tops)


def centroids(seed: int, layer: int, G: int, d: int) -> np.ndarray:
    return _rng(seed, 0xCE27, layer).standard_normal((G, N_TOPICS, d)).astype(np.float32)


def kv_layer(seed: int, layer: int, topics: np.ndarray, G: int, d: int):
    """K, V bf16 bits [B][G][L][d] for one layer."""
    B, L = topics.shape
    c = centroids(seed, layer, G, d)
    rng = _rng(seed, 0x4B56, layer)
    K = np.empty((B, G, L, d), dtype=np.uint16)
    V = np.empty((B, G, L, d), dtype=np.uint16)
    for b in range(B):
        for g in range(G):
            K[b, g] = f32_to_bf16_bits(c[g][topics[b]] + rng.standard_normal((L, d), dtype=np.float32))
            V[b, g] = f32_to_bf16_bits(rng.standard_normal((L, d), dtype=np.float32))
    return K, V


def decode_script(seed: int, B: int, steps: int, boundary_ids=BOUNDARY_IDS, mean_sentence: float = 25.0):
    """Per step: input token ids [steps][B] and the target topic of each step [steps][B].

    The generated text of each sequence is a run of sentences whose lengths follow the prompt's
    distribution (lognormal, median `mean_sentence`, clamp [2, 256]); the last token of each sentence
    is a boundary id, after which the target topic changes.  The first sentence of each sequence
    starts at a random phase, so the sequences' boundaries are staggered."""
    rng = _rng(seed, 0xDEC0)
    bset = np.asarray(boundary_ids, dtype=np.int32)
    is_b = np.zeros((steps, B), dtype=bool)
    for b in range(B):
        n = np.clip(np.rint(np.exp(rng.normal(np.log(mean_sentence), 0.5, size=steps + 2))), 2, 256).astype(np.int64)
        ends = np.cumsum(n) - 1 - int(rng.integers(0, n[0]))
        ends = ends[(ends >= 0) & (ends < steps)]
        is_b[ends, b] = True
    tok = rng.integers(VOCAB_LO, VOCAB_HI, size=(steps, B)).astype(np.int32)
    tok = np.where(np.isin(tok, bset), VOCAB_LO, tok).astype(np.int32)
    tok[is_b] = bset[rng.integers(0, len(bset), size=int(is_b.sum()))]
    target = np.zeros((steps, B), dtype=np.int32)
    cur = rng.integers(0, N_TOPICS, size=B)
    for t in range(steps):
        target[t] = cur
        nxt = rng.integers(0, N_TOPICS, size=B)
        cur = np.where(is_b[t], nxt, cur)
    return tok, target


def queries(seed: int, layer: int, step: int, target: np.ndarray, Hq: int, G: int, d: int) -> np.ndarray:
    """q_t bf16 bits [B][Hq][d] for one (layer, step)."""
    c = centroids(seed, layer, G, d)
    grp = Hq // G
    rng = _rng(seed, 0x9E11, layer, step)
    B = target.shape[0]
    q = np.empty((B, Hq, d), dtype=np.float32)
    for b in range(B):
        for h in range(Hq):
            q[b, h] = c[h // grp, target[b]] + rng.standard_normal(d, dtype=np.float32)
    return f32_to_bf16_bits(q)


# ------------------------------------------------------------- GPU-side generation (bench)


def kv_layer_torch(seed: int, layer: int, topics, G: int, d: int, device="cuda", b_begin: int = 0,
                   g_begin: int = 0, g_count: int = None):
    """Same recipe as kv_layer, drawn on the GPU with seeded torch generators (for the full-size
    bench configs where numpy generation would take minutes).  topics: int tensor [B_loc][L] of the
    global sequences b_begin .. b_begin + B_loc; returns bf16 K, V [B_loc][g_count][L][d] for KV
    heads g_begin .. g_begin + g_count and the layer's centroids [G][T][d].  Every (layer, b, g)
    has its own generator, so any shard layout draws the same numbers."""
    import torch

    g_count = G - g_begin if g_count is None else g_count
    gen = torch.Generator(device=device)
    gen.manual_seed((seed * 1_000_003 + layer * 7919 + 0xCE27) & 0x7FFFFFFFFFFFFFFF)
    c = torch.randn((G, N_TOPICS, d), generator=gen, device=device, dtype=torch.float32)
    B, L = topics.shape
    K = torch.empty((B, g_count, L, d), dtype=torch.bfloat16, device=device)
    V = torch.empty((B, g_count, L, d), dtype=torch.bfloat16, device=device)
    tl = topics.long()
    for bi in range(B):
        for gi in range(g_count):
            b, g = b_begin + bi, g_begin + gi
            gen.manual_seed((seed * 1_000_003 + layer * 7919 + b * 131 + g * 17 + 0x4B56) & 0x7FFFFFFFFFFFFFFF)
            K[bi, gi] = (c[g][tl[bi]] + torch.randn((L, d), generator=gen, device=device)).to(torch.bfloat16)
            V[bi, gi] = torch.randn((L, d), generator=gen, device=device).to(torch.bfloat16)
    return K, V, c


def queries_torch(gen, centroids_g, target, Hq: int, G: int, d: int):
    """q_t bf16 [B][Hq][d] = centroid of the target topic (per KV head group) + N(0, 1)."""
    import torch

    grp = Hq // G
    B = target.shape[0]
    c = centroids_g[:, target.long(), :]                  # [G][B][d]
    c = c.permute(1, 0, 2).repeat_interleave(grp, dim=1)  # [B][Hq][d]
    return (c + torch.randn((B, Hq, d), generator=gen, device=c.device)).to(torch.bfloat16)


def window_queries(seed: int, layer: int, target: np.ndarray, Hq: int, G: int, d: int, scale: float = 1.0) -> np.ndarray:
    """NEXT-1 observation-window queries: bf16 bits [B][N][Hq][d], row w of sequence b
    = scale * c[layer, g(h), target[b][w]] + N(0, 1).  target = the topics of the last N prompt
    tokens (the window asks about its own content), or any topics a test wants to emphasise."""
    c = centroids(seed, layer, G, d)
    grp = Hq // G
    rng = _rng(seed, 0x0B5E, layer)
    B, N = target.shape
    q = np.empty((B, N, Hq, d), dtype=np.float32)
    for b in range(B):
        for w in range(N):
            for h in range(Hq):
                q[b, w, h] = scale * c[h // grp, target[b, w]] + rng.standard_normal(d, dtype=np.float32)
    return f32_to_bf16_bits(q)


def window_queries_torch(gen, centroids_g, target, Hq: int, G: int, d: int, scale: float = 1.0):
    """GPU twin of window_queries for the full-size bench: bf16 [B][N][Hq][d] from the layer's
    centroids [G][T][d] and the target topics [B][N] (seeded torch generator)."""
    import torch

    grp = Hq // G
    c = centroids_g[:, target.long(), :]                      # [G][B][N][d]
    c = c.permute(1, 2, 0, 3).repeat_interleave(grp, dim=2)   # [B][N][Hq][d]
    return (scale * c + torch.randn(c.shape, generator=gen, device=c.device)).to(torch.bfloat16)
