"""Pins for the oracle's D2 selection, D4 attention (Eq. 3), the Algorithm 1
driver and the memory accounting -- CPU only."""
import os

import numpy as np
import pytest
import torch

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden", "selection.txt")


def bits(x):
    return synth.f32_to_bf16_bits(np.asarray(x, np.float32))


def f32(h):
    return synth.bf16_bits_to_f32(h)


def off_of(lengths):
    return np.concatenate([[0], np.cumsum(lengths)]).astype(np.int32)


# ----------------------------------------------------------------------------- selection


def _golden():
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        sid, tau, lens, scores, ids, ntok = (x.strip() for x in line.split("|"))
        yield (sid, int(tau), [int(v) for v in lens.split()], [float(v) for v in scores.split()],
               [int(v) for v in ids.split()], int(ntok))


@pytest.mark.parametrize("sid,tau,lens,scores,want_ids,want_ntok", list(_golden()))
def test_select_worked(sid, tau, lens, scores, want_ids, want_ntok):
    ids, ntok = oracle.select(np.array(scores, np.float32), off_of(lens), tau)
    assert ids.tolist() == want_ids and ntok == want_ntok, sid


def _brute_force(scores, lens, tau):
    """The unique subset that (i) fits tau, (ii) is upward-closed in (score desc, index asc)
    order, (iii) is maximal -- found by enumerating all 2^S subsets."""
    S = len(scores)
    sc = [0.0 if x == 0 else x for x in scores]  # -0 == +0

    def better(a, b):  # a ranks before b
        if np.isnan(sc[a]):
            return False if not np.isnan(sc[b]) else a < b
        if np.isnan(sc[b]):
            return True
        return sc[a] > sc[b] or (sc[a] == sc[b] and a < b)

    best = None
    for mask in range(1 << S):
        sub = [s for s in range(S) if mask >> s & 1]
        if sum(lens[s] for s in sub) > tau:
            continue
        # upward closed: every sentence ranked before a member is a member
        if any(better(o, s) and o not in sub for s in sub for o in range(S)):
            continue
        if best is None or len(sub) > len(best):
            best = sub
    return best


@pytest.mark.parametrize("seed", range(40))
def test_select_equals_brute_force(seed):
    rng = np.random.default_rng(seed)
    S = int(rng.integers(1, 13))
    lens = rng.integers(1, 9, size=S).tolist()
    # few distinct values so that ties are frequent
    scores = rng.choice(np.array([-1.0, -0.0, 0.0, 0.5, 0.5, 2.0, np.nan], np.float32), size=S)
    tau = int(rng.integers(1, 30))
    ids, ntok = oracle.select(scores, off_of(lens), tau)
    want = _brute_force(scores.tolist(), lens, tau)
    assert ids.tolist() == sorted(want)
    assert ntok == sum(lens[s] for s in want) <= tau


def test_zero_query_selects_document_prefix():
    # q = 0 => all scores +0 => ties => sentences in document order until tau
    toks, topics = synth.prompts(1, 1, 4096, median=20.0)
    off = oracle.segment(toks[0], synth.BOUNDARY_IDS, 256)
    K, _ = synth.kv_layer(1, 0, topics, 1, 64)
    E = oracle.embed(K[0, 0], off)
    sc = oracle.score(np.zeros(64, np.float32), E)
    ids, ntok = oracle.select(sc, off, 256)
    k = int(np.searchsorted(off, 256, side="right")) - 1  # sentences [0, k) fit
    assert ids.tolist() == list(range(k)) and ntok == off[k]


def test_budget_covers_everything_selects_all():
    lens = [3, 1, 4, 1, 5]
    ids, ntok = oracle.select(np.array([1, 5, 2, 4, 3], np.float32), off_of(lens), 14)
    assert ids.tolist() == [0, 1, 2, 3, 4] and ntok == 14


# ----------------------------------------------------------------------------- attention


def test_attend_single_token_returns_its_value():
    rng = np.random.default_rng(0)
    q, K, V = bits(rng.standard_normal((4, 64))), bits(rng.standard_normal((9, 64))), bits(rng.standard_normal((9, 64)))
    off = off_of([3, 1, 5])
    O = oracle.attend(q, K, V, off, np.array([1], np.int32))
    assert np.allclose(O, np.tile(f32(V[3]), (4, 1)), rtol=0, atol=1e-15)


def test_attend_identical_keys_gives_mean_value():
    rng = np.random.default_rng(1)
    K = np.tile(bits(rng.standard_normal(64)), (6, 1))
    V = bits(rng.standard_normal((6, 64)))
    q = bits(rng.standard_normal((2, 64)))
    O = oracle.attend(q, K, V, off_of([6]), np.array([0], np.int32))
    assert np.allclose(O, np.tile(f32(V).astype(np.float64).mean(0), (2, 1)), atol=1e-14)


@pytest.mark.parametrize("d,grp", [(64, 4), (128, 1), (128, 8)])
def test_attend_matches_torch_sdpa_fp64(d, grp):
    rng = np.random.default_rng(d + grp)
    L = 300
    q = bits(rng.standard_normal((grp, d)) * 2)
    K = bits(rng.standard_normal((L, d)) * 2)
    V = bits(rng.standard_normal((L, d)))
    lens = [7, 13, 40, 1, 100, 139]
    off = off_of(lens)
    ids = np.array([1, 3, 4], np.int32)
    rows = np.concatenate([np.arange(off[s], off[s + 1]) for s in ids])
    t = lambda a: torch.from_numpy(f32(a).astype(np.float64))
    ref = torch.nn.functional.scaled_dot_product_attention(
        t(q)[None, :, None, :], t(K[rows])[None, None].expand(1, grp, -1, -1), t(V[rows])[None, None].expand(1, grp, -1, -1)
    )[0, :, 0, :].numpy()
    O = oracle.attend(q, K, V, off, ids)
    assert np.max(np.abs(O - ref)) < 1e-12


def test_full_budget_pipeline_equals_full_attention():
    """tau >= L  =>  every sentence is selected  =>  Eq. 3 == full attention (P:614 Full KV,
    SPEC acceptance criterion 1), checked against torch's fp64 SDPA."""
    B, L, G, Hq, d, M = 2, 512, 2, 8, 64, 2
    toks, topics = synth.prompts(7, B, L, median=20.0)
    orc = oracle.Oracle(toks, synth.BOUNDARY_IDS, tau=L, layers=M, q_heads=Hq, kv_heads=G, d=d)
    script_tok, target = synth.decode_script(7, B, 3)
    for l in range(M):
        K, V = synth.kv_layer(7, l, topics, G, d)
        orc.prefill_layer(l, K, V)
    for step in range(3):
        for l in range(M):
            q = synth.queries(7, l, step, target[step], Hq, G, d)
            _, ids, ntok = orc.decode_select(l, q, script_tok[step])
            O = orc.decode_attend(l, q, ids)
            t = lambda a: torch.from_numpy(f32(a).astype(np.float64))
            for b in range(B):
                for g in range(G):
                    assert ntok[b][g] == L and len(ids[b][g]) == len(orc.off[b]) - 1
                    hs = slice(g * Hq // G, (g + 1) * Hq // G)
                    ref = torch.nn.functional.scaled_dot_product_attention(
                        t(q[b, hs])[:, None, :], t(orc.K[l][b, g])[None], t(orc.V[l][b, g])[None]
                    )[:, 0, :].numpy()
                    assert np.max(np.abs(O[b, hs] - ref)) < 1e-12


def test_pipeline_budget_law_and_reset_count():
    B, L, G, Hq, d, tau = 1, 4096, 2, 8, 64, 256
    toks, topics = synth.prompts(3, B, L, median=20.0)
    orc = oracle.Oracle(toks, synth.BOUNDARY_IDS, tau=tau, layers=1, q_heads=Hq, kv_heads=G, d=d)
    K, V = synth.kv_layer(3, 0, topics, G, d)
    orc.prefill_layer(0, K, V)
    steps = 60
    script_tok, target = synth.decode_script(3, B, steps)
    resets = 0
    for step in range(steps):
        q = synth.queries(3, 0, step, target[step], Hq, G, d)
        _, ids, ntok = orc.decode_select(0, q, script_tok[step])
        n = orc.off[0]
        for g in range(G):
            assert ntok[0][g] == sum(int(n[s + 1] - n[s]) for s in ids[0][g]) <= tau
        if script_tok[step, 0] in synth.BOUNDARY_IDS:
            resets += 1
            assert orc.cnt[0, 0] == 0
    assert resets == int(np.isin(script_tok[:, 0], synth.BOUNDARY_IDS).sum()) > 0


def test_selection_prefers_the_query_topic():
    """q built from one topic's centroid => the top-ranked sentences share that topic (the
    similarity mechanism of P:440-444 on the synthetic topic model)."""
    B, L, G, Hq, d, tau = 1, 4096, 1, 4, 64, 128
    toks, topics = synth.prompts(5, B, L, median=20.0)
    orc = oracle.Oracle(toks, synth.BOUNDARY_IDS, tau=tau, layers=1, q_heads=Hq, kv_heads=G, d=d)
    K, V = synth.kv_layer(5, 0, topics, G, d)
    orc.prefill_layer(0, K, V)
    target = np.array([topics[0, 100]], np.int32)
    q = synth.queries(5, 0, 0, target, Hq, G, d)
    _, ids, _ = orc.decode_select(0, q, np.array([500], np.int32))
    off = orc.off[0]
    on_topic = [s for s in range(len(off) - 1) if topics[0, off[s]] == target[0]]
    assert sum(int(off[s + 1] - off[s]) for s in on_topic) <= tau  # they all fit ...
    assert set(on_topic) <= set(ids[0][0].tolist())  # ... and are all retrieved


# ----------------------------------------------------------------------------- accounting


def test_kv_bytes_paper_numbers():
    # "processing a 32k-token prompt ... requires approximately 16 GB (using float16)",
    # with the Cost(t) formula of P:563 (M=32 layers, H=32 heads, d=128).
    assert oracle.kv_bytes(32, 32, 128, 32768) == 17_179_869_184 == 16 * 2**30
    # 256K (= 256,000 tokens) Llama-3.1-8B KV cache: 33.55 GB: 8 KV heads (GQA)
    assert round(oracle.kv_bytes(32, 8, 128, 256_000) / 1e9, 2) == 33.55
    assert oracle.kv_bytes(32, 8, 128, 0) == 0
