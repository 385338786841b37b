"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same seeded inputs.

Bars (north_star): segmentation offsets, sentence embeddings, scores and selected
sentence ids / counts / token counts bit-exact; attention output max-abs <= 2e-3 vs the fp64
oracle on the same selection.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests.gpu_harness import ATOL, from_bits, make_case, run_parity, to_bits

pytestmark = pytest.mark.gpu


def _skv(B, M, Hq, G, d, L, tau, **kw):
    import paper_2504_00970_b200 as skvlib

    return skvlib.SentenceKV(batch=B, layers=M, q_heads=Hq, kv_heads=G, head_dim=d, max_context=L,
                             token_budget=tau, **kw)


@pytest.mark.parametrize("mode", ["split", "step"])
@pytest.mark.parametrize("seed", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("Hq", [8, 2])
def test_tiny_config_full_parity(cuda_device, seed, Hq, mode):
    """configs[0]: 1 layer, 2 KV heads, d=64, 4K tokens, ~20-token sentences, tau=256, B=1
    (Hq=8 -> GQA grp=4; Hq=2 -> MHA)."""
    B, M, G, d, L, tau, steps = 1, 1, 2, 64, 4096, 256, 40
    toks, _, Ks, Vs, qs, script = make_case(seed, B, M, Hq, G, d, L, tau, steps, median=20.0)
    skv = _skv(B, M, Hq, G, d, L, tau)
    orc = oracle.Oracle(toks, synth.BOUNDARY_IDS, tau, M, Hq, G, d)
    st = run_parity(skv, orc, toks, Ks, Vs, qs, script, synth.BOUNDARY_IDS, cuda_device, mode=mode)
    assert st["steps"] == steps and st["max_abs"] <= ATOL


@pytest.mark.parametrize("mode", ["split", "step"])
def test_multi_sequence_multi_layer_gqa8(cuda_device, mode):
    """B=3 prompts of different sentence counts, 2 layers, grp=8 (70B-style), d=128, ragged L."""
    B, M, Hq, G, d, L, tau, steps = 3, 2, 16, 2, 128, 5003, 512, 12
    toks, _, Ks, Vs, qs, script = make_case(11, B, M, Hq, G, d, L, tau, steps, median=25.0)
    skv = _skv(B, M, Hq, G, d, L, tau)
    orc = oracle.Oracle(toks, synth.BOUNDARY_IDS, tau, M, Hq, G, d)
    run_parity(skv, orc, toks, Ks, Vs, qs, script, synth.BOUNDARY_IDS, cuda_device, mode=mode)


@pytest.mark.parametrize("mode", ["split", "step"])
def test_llama8b_32k_config(cuda_device, mode):
    """configs[1] shapes (8 KV / 32 Q heads, d=128, 32K context, tau=1024, B=1) on 2 of the 32
    layers, every (b, g) unit, 6 decode steps."""
    B, M, Hq, G, d, L, tau, steps = 1, 2, 32, 8, 128, 32768, 1024, 6
    toks, _, Ks, Vs, qs, script = make_case(5, B, M, Hq, G, d, L, tau, steps, median=25.0)
    skv = _skv(B, 32, Hq, G, d, L, tau)  # ctx for all 32 layers; 2 exercised
    orc = oracle.Oracle(toks, synth.BOUNDARY_IDS, tau, M, Hq, G, d)
    run_parity(skv, orc, toks, Ks, Vs, qs, script, synth.BOUNDARY_IDS, cuda_device, mode=mode)


def test_budget_at_least_context_equals_full_attention(cuda_device):
    """tau >= L: every sentence is selected and Eq. 3 equals full attention (O-FULL)."""
    B, M, Hq, G, d, L, tau = 2, 1, 8, 2, 128, 1500, 1500
    toks, _, Ks, Vs, qs, script = make_case(3, B, M, Hq, G, d, L, tau, 3, median=25.0)
    skv = _skv(B, M, Hq, G, d, L, tau)
    orc = oracle.Oracle(toks, synth.BOUNDARY_IDS, tau, M, Hq, G, d)
    st = run_parity(skv, orc, toks, Ks, Vs, qs, script, synth.BOUNDARY_IDS, cuda_device)
    assert all(t == L for t in st["sel_tokens"])
    # and against torch's fp64 SDPA over all L tokens
    out = torch.empty((B, Hq, d), dtype=torch.float32, device=cuda_device)
    qd = from_bits(qs[-1][0], cuda_device)
    skv.decode_attend(0, qd, out)
    K = torch.from_numpy(synth.bf16_bits_to_f32(Ks[0]).astype(np.float64))
    V = torch.from_numpy(synth.bf16_bits_to_f32(Vs[0]).astype(np.float64))
    q = torch.from_numpy(synth.bf16_bits_to_f32(qs[-1][0]).astype(np.float64))
    grp = Hq // G
    ref = torch.nn.functional.scaled_dot_product_attention(
        q.view(B, G, grp, d), K, V)  # [B][G][grp][d]
    assert float((out.cpu().double().view(B, G, grp, d) - ref).abs().max()) <= ATOL


# --------------------------------------------------------------------------- edge cases


def _custom_case(device, toks, K_bits, V_bits, q_list, script, tau, Hq, G, d, bset=synth.BOUNDARY_IDS):
    """Runs the case through both the split calls and the fused decode_step."""
    B, L = toks.shape
    for mode in ("split", "step"):
        skv = _skv(B, 1, Hq, G, d, L, tau)
        orc = oracle.Oracle(toks, bset, tau, 1, Hq, G, d)
        st = run_parity(skv, orc, toks, [K_bits], [V_bits], [[q] for q in q_list], script, bset, device, mode=mode)
    return st


def test_ties_duplicated_sentences_and_zero_query(cuda_device):
    """Tie stress: duplicated sentences (identical E -> equal scores, lowest index first) and
    q = 0 (all scores +0 -> document order)."""
    B, Hq, G, d, L, tau = 1, 4, 1, 64, 2000, 200
    toks, topics = synth.prompts(21, B, L, median=20.0)
    K, V = synth.kv_layer(21, 0, topics, G, d)
    off = oracle.segment(toks[0], synth.BOUNDARY_IDS, tau)
    lens = np.diff(off)
    # copy sentence 3's keys over every later sentence of the same length
    for s in range(4, len(lens)):
        if lens[s] == lens[3]:
            K[0, 0, off[s]:off[s + 1]] = K[0, 0, off[3]:off[4]]
    rng = np.random.default_rng(0)
    e3 = synth.bf16_bits_to_f32(K[0, 0, off[3]:off[4]]).mean(0)
    q_dup = synth.f32_to_bf16_bits(np.tile(e3 * 3, (B, Hq, 1)))
    q_zero = np.zeros((B, Hq, d), np.uint16)
    q_rand = synth.f32_to_bf16_bits(rng.standard_normal((B, Hq, d)).astype(np.float32))
    script = np.array([[500], [13], [500], [500]], np.int32)  # reset after step 1
    _custom_case(cuda_device, toks, K, V, [q_dup, q_zero, q_zero, q_rand], script, tau, Hq, G, d)


def test_all_equal_keys(cuda_device):
    B, Hq, G, d, L, tau = 2, 8, 2, 128, 777, 64
    toks, _ = synth.prompts(4, B, L, median=20.0)
    k = synth.f32_to_bf16_bits(np.random.default_rng(1).standard_normal(d).astype(np.float32))
    K = np.broadcast_to(k, (B, G, L, d)).copy()
    V = synth.f32_to_bf16_bits(np.random.default_rng(2).standard_normal((B, G, L, d)).astype(np.float32))
    qs = [synth.f32_to_bf16_bits(np.random.default_rng(3 + i).standard_normal((B, Hq, d)).astype(np.float32))
          for i in range(3)]
    _custom_case(cuda_device, toks, K, V, qs, np.full((3, B), 300, np.int32), tau, Hq, G, d)


@pytest.mark.parametrize("L,tau", [(1, 16), (5, 16), (64, 64), (65, 64), (300, 64), (1000, 1)])
def test_tau_cap_and_tiny_prompts(cuda_device, L, tau):
    """Sentences of exactly tau and tau+1 tokens (tau-cap, A5), L = 1, a single sentence, tau = 1."""
    B, Hq, G, d = 1, 4, 1, 64
    rng = np.random.default_rng(L * 7 + tau)
    toks = rng.integers(256, 128000, size=(B, L)).astype(np.int32)
    # boundaries at a few fixed places so that runs of exactly tau and tau+1 occur
    for p in (tau - 1, 2 * tau, 3 * tau + 1):
        if p < L:
            toks[0, p] = synth.BOUNDARY_IDS[0]
    K = synth.f32_to_bf16_bits(rng.standard_normal((B, G, L, d)).astype(np.float32))
    V = synth.f32_to_bf16_bits(rng.standard_normal((B, G, L, d)).astype(np.float32))
    qs = [synth.f32_to_bf16_bits(rng.standard_normal((B, Hq, d)).astype(np.float32)) for _ in range(3)]
    _custom_case(cuda_device, toks, K, V, qs, np.full((3, B), 300, np.int32), tau, Hq, G, d)


def test_many_one_token_sentences(cuda_device):
    """Every token a boundary: S = L one-token sentences (max sentence count)."""
    B, Hq, G, d, L, tau = 1, 8, 2, 64, 3000, 100
    toks = np.full((B, L), synth.BOUNDARY_IDS[1], np.int32)
    rng = np.random.default_rng(9)
    K = synth.f32_to_bf16_bits(rng.standard_normal((B, G, L, d)).astype(np.float32))
    V = synth.f32_to_bf16_bits(rng.standard_normal((B, G, L, d)).astype(np.float32))
    qs = [synth.f32_to_bf16_bits(rng.standard_normal((B, Hq, d)).astype(np.float32)) for _ in range(2)]
    _custom_case(cuda_device, toks, K, V, qs, np.full((2, B), 300, np.int32), tau, Hq, G, d)


@pytest.mark.parametrize("L", [3000, 12000])
def test_one_token_sentences_zero_query(cuda_device, L):
    """q = 0 on one-token sentences: every score ties at +0, so the one-launch step kernel keeps every
    sentence as a local candidate (L = 12000: lists overflow shared memory into the global scratch
    and the union is ranked in place); the selection must still be the first tau sentences."""
    B, Hq, G, d, tau = 1, 8, 2, 64, 100
    toks = np.full((B, L), synth.BOUNDARY_IDS[2], np.int32)
    rng = np.random.default_rng(L)
    K = synth.f32_to_bf16_bits(rng.standard_normal((B, G, L, d)).astype(np.float32))
    V = synth.f32_to_bf16_bits(rng.standard_normal((B, G, L, d)).astype(np.float32))
    q0 = np.zeros((B, Hq, d), np.uint16)
    q1 = synth.f32_to_bf16_bits(rng.standard_normal((B, Hq, d)).astype(np.float32))
    _custom_case(cuda_device, toks, K, V, [q0, q0, q1], np.array([[300], [13], [300]], np.int32), tau, Hq, G, d)


@pytest.mark.parametrize("band_log2", ["0", "12", "29"])
def test_step_kernel_selection_paths_subprocess(cuda_device, band_log2):
    """The one-launch step kernel ranks either the band around the previous crossing point or, when
    the crossing left the band, the entries above it (mode 2) or the union of the local candidate
    lists (general path).  A narrow band (sentencekv_set_band_log2 0 or 12, applied to every context of
    the child pytest by tests/conftest.py) sends most steps through mode 2 and the general path, a very
    wide one (29) overflows the band lists: all must give the oracle's selections and outputs."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, SKV_TEST_BAND_LOG2=band_log2)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-x", "tests/test_gpu_parity.py",
                        "tests/test_gpu_fullsize.py",
                        "-k", "(step or ties or all_equal or one_token or config2) and not subprocess"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("residency", ["device", "host"])
def test_graph_replay_parity(cuda_device, residency):
    """bench.py's launch configuration: the decode step of all layers captured once into a CUDA graph
    (programmatic launch between the layers' kernels) and replayed for every step with new inputs;
    the device-side state (selection slot parity, band hints, Q_s sums, page cache) must evolve as
    in the oracle, step after step."""
    import paper_2504_00970_b200 as skvlib

    B, M, Hq, G, d, L, tau, steps = 2, 3, 16, 4, 128, 8192, 512, 6
    toks, topics, Ks, Vs, qs, script = make_case(3, B, M, Hq, G, d, L, tau, steps, 25.0)
    skv = _skv(B, M, Hq, G, d, L, tau,
               residency=skvlib.SKV_KV_HOST if residency == "host" else skvlib.SKV_KV_DEVICE)
    orc = oracle.Oracle(toks, synth.BOUNDARY_IDS, tau, M, Hq, G, d)
    st = run_parity(skv, orc, toks, Ks, Vs, qs, script, synth.BOUNDARY_IDS, cuda_device, mode="graph")
    assert st["steps"] == steps


@pytest.mark.parametrize("mode", ["split", "step"])
def test_deterministic_run_to_run(cuda_device, mode):
    """Two runs of the same inputs give bit-identical selections and outputs (static work split,
    fixed merge order; no atomics decide an fp32 summation order)."""
    B, M, Hq, G, d, L, tau, steps = 2, 1, 8, 2, 128, 6000, 512, 5
    toks, _, Ks, Vs, qs, script = make_case(8, B, M, Hq, G, d, L, tau, steps, median=25.0)
    outs = []
    for _ in range(2):
        skv = _skv(B, M, Hq, G, d, L, tau)
        tok_dev = torch.from_numpy(toks).to(cuda_device)
        skv.prefill_compress(0, from_bits(Ks[0], cuda_device), from_bits(Vs[0], cuda_device), tok_dev,
                             synth.BOUNDARY_IDS)
        ids = torch.empty((B, G, tau), dtype=torch.int32, device=cuda_device)
        out = torch.empty((B, Hq, d), dtype=torch.float32, device=cuda_device)
        res = []
        for s in range(steps):
            qd = from_bits(qs[s][0], cuda_device)
            it = torch.from_numpy(script[s]).to(cuda_device)
            if mode == "step":
                skv.decode_step(0, qd, it, out, ids)
            else:
                skv.decode_select(0, qd, it, ids)
                skv.decode_attend(0, qd, out)
            res.append((ids.cpu().numpy().copy(), out.cpu().numpy().copy()))
        outs.append(res)
    for (i1, o1), (i2, o2) in zip(*outs):
        assert np.array_equal(i1, i2) and np.array_equal(o1.view(np.uint32), o2.view(np.uint32))


# --------------------------------------------------------------------------- host residency (P3 + D3)


@pytest.mark.parametrize("mode", ["split", "step"])
@pytest.mark.parametrize("seed,Hq,G,d,B,L,tau,median", [
    (0, 8, 2, 64, 1, 4096, 256, 20.0),      # configs[0] shapes
    (11, 16, 2, 128, 3, 5003, 512, 25.0),   # ragged, grp = 8
])
def test_host_residency_parity(cuda_device, mode, seed, Hq, G, d, B, L, tau, median):
    """Full K/V offloaded to pinned host (P3); each step gathers from the HBM working set (previous
    selection) and from host memory (misses).  Results must equal the oracle exactly as in device
    residency: any stale working-set row or bad host fetch shows up in O."""
    import paper_2504_00970_b200 as skvlib

    M, steps = 2, 30
    toks, _, Ks, Vs, qs, script = make_case(seed, B, M, Hq, G, d, L, tau, steps, median=median)
    skv = _skv(B, M, Hq, G, d, L, tau, residency=skvlib.SKV_KV_HOST)
    orc = oracle.Oracle(toks, synth.BOUNDARY_IDS, tau, M, Hq, G, d)
    st = run_parity(skv, orc, toks, Ks, Vs, qs, script, synth.BOUNDARY_IDS, cuda_device, mode=mode)
    assert st["max_abs"] <= ATOL


def test_host_residency_transfer_ledger(cuda_device):
    """Ledger pins (SURVEY 8(c) D3 host): the first step fetches every
    selected byte from host memory; repeating the same query (no boundary) leaves the selection
    unchanged, so the next step fetches 0 bytes; a different topic fetches some."""
    import paper_2504_00970_b200 as skvlib

    B, Hq, G, d, L, tau = 2, 8, 2, 128, 6000, 512
    toks, topics = synth.prompts(2, B, L, median=25.0)
    K, V = synth.kv_layer(2, 0, topics, G, d)
    skv = _skv(B, 1, Hq, G, d, L, tau, residency=skvlib.SKV_KV_HOST)
    skv.prefill_compress(0, from_bits(K, cuda_device), from_bits(V, cuda_device),
                         torch.from_numpy(toks).to(cuda_device), synth.BOUNDARY_IDS)
    tgt = np.array([3, 9], np.int32)
    q1 = from_bits(synth.queries(2, 0, 0, tgt, Hq, G, d), cuda_device)
    q2 = from_bits(synth.queries(2, 0, 1, (tgt + 20) % synth.N_TOPICS, Hq, G, d), cuda_device)
    no_b = torch.full((B,), 300, dtype=torch.int32, device=cuda_device)
    ntok = torch.empty((B, G), dtype=torch.int32, device=cuda_device)
    out = torch.empty((B, Hq, d), dtype=torch.float32, device=cuda_device)
    row = d * 2 * 2  # K + V bytes per token
    skv.decode_step(0, q1, no_b, out, sel_tokens=ntok)
    first = skv.host_fetch_bytes(0)
    assert first == int(ntok.sum()) * row > 0
    ids1 = torch.empty((B, G, tau), dtype=torch.int32, device=cuda_device)
    skv.decode_step(0, q1, no_b, out, sel_ids=ids1)  # qbar = (q1 + q1) / 2 = q1: same selection
    assert skv.host_fetch_bytes(0) == first
    reset = torch.full((B,), int(synth.BOUNDARY_IDS[0]), dtype=torch.int32, device=cuda_device)
    skv.decode_step(0, q1, reset, out)  # still q1; resets Q_s afterwards
    assert skv.host_fetch_bytes(0) == first
    skv.decode_step(0, q2, no_b, out, sel_tokens=ntok)  # qbar = q2 (fresh sentence): new topic
    assert skv.host_fetch_bytes(0) > first


def test_host_residency_drift_fetches_each_row_once(cuda_device):
    """Drift within a topic (Q_s grows, qbar moves, sentences enter the selection step by step): with a
    page cache large enough to hold every selection of the run (r = 8), each step fetches from host
    exactly the rows of its selection never selected before -- rows that enter a page already holding
    a slot (filled in without a cache plan) or a page reserved for the sentences just below the
    crossing point (slot, no rows) included: nothing is fetched twice, nothing unselected is fetched.
    Selected ids equal the oracle's at every step."""
    import paper_2504_00970_b200 as skvlib

    B, Hq, G, d, L, tau, steps = 2, 8, 2, 64, 6000, 256, 12
    toks, topics = synth.prompts(5, B, L, median=12.0)
    K, V = synth.kv_layer(5, 0, topics, G, d)
    skv = _skv(B, 1, Hq, G, d, L, tau, residency=skvlib.SKV_KV_HOST, semantic_factor=8.0)
    orc = oracle.Oracle(toks, synth.BOUNDARY_IDS, tau, 1, Hq, G, d)
    skv.prefill_compress(0, from_bits(K, cuda_device), from_bits(V, cuda_device),
                         torch.from_numpy(toks).to(cuda_device), synth.BOUNDARY_IDS)
    orc.prefill_layer(0, K, V)
    off = skv.offsets().cpu().numpy()
    tgt = np.array([4, 11], np.int32)
    no_b = np.full((B,), 300, np.int32)
    ids = torch.empty((B, G, tau), dtype=torch.int32, device=cuda_device)
    out = torch.empty((B, Hq, d), dtype=torch.float32, device=cuda_device)
    seen = [[set() for _ in range(G)] for _ in range(B)]
    row = d * 2 * 2  # K + V bytes per token
    changed = 0
    for s in range(steps):
        q = synth.queries(5, 0, s, tgt, Hq, G, d)
        before = skv.host_fetch_bytes(0)
        skv.decode_step(0, from_bits(q, cuda_device), torch.from_numpy(no_b).to(cuda_device), out, sel_ids=ids)
        _, ids_o, _ = orc.decode_select(0, q, no_b)
        got = ids.cpu().numpy()
        expect = 0
        for b in range(B):
            for g in range(G):
                n = len(ids_o[b][g])
                assert np.array_equal(got[b, g, :n], ids_o[b][g]), f"ids s={s} b={b} g={g}"
                rows = set()
                for sid in ids_o[b][g]:
                    rows.update(range(int(off[b, sid]), int(off[b, sid + 1])))
                new = rows - seen[b][g]
                changed += 1 if (s > 0 and new) else 0
                expect += len(new) * row
                seen[b][g] |= rows
        assert skv.host_fetch_bytes(0) - before == expect, f"step {s}"
    assert changed >= 2  # the selection did drift


@pytest.mark.parametrize("mode", ["split", "step"])
@pytest.mark.parametrize("L,tau,median", [
    (40000, 4096, 25.0),   # configs[3]'s budget: ~400 pages of 16 rows per selection
    (12000, 2048, 3.0),    # short sentences: a selection touches ~1000 pages
])
def test_host_residency_large_selections(cuda_device, mode, L, tau, median):
    """Host residency with selections spanning more pages than the step kernel's cache plan tracks
    (pages past the plan must never be evicted while they are read): selections and
    outputs equal the oracle over topic switches."""
    import paper_2504_00970_b200 as skvlib

    B, M, Hq, G, d, steps = 1, 1, 8, 2, 128, 16
    toks, _, Ks, Vs, qs, script = make_case(21, B, M, Hq, G, d, L, tau, steps, median=median)
    skv = _skv(B, M, Hq, G, d, L, tau, residency=skvlib.SKV_KV_HOST)
    orc = oracle.Oracle(toks, synth.BOUNDARY_IDS, tau, M, Hq, G, d)
    st = run_parity(skv, orc, toks, Ks, Vs, qs, script, synth.BOUNDARY_IDS, cuda_device, mode=mode)
    assert st["max_abs"] <= ATOL


@pytest.mark.parametrize("mode", ["split", "step"])
def test_nan_inf_and_signed_zero_keys(cuda_device, mode):
    """The key rule on the GPU (reading A14: NaN scores rank last, -0 == +0, +-Inf order as numbers):
    sentences whose keys hold NaN, +Inf or -Inf give NaN / infinite embeddings and scores; the scores
    (bit patterns) and the selected ids must equal the oracle's, and O where both sides are finite."""
    import paper_2504_00970_b200 as skvlib

    B, Hq, G, d, L, tau, steps = 1, 4, 1, 64, 3000, 120, 6
    toks, topics = synth.prompts(31, B, L, median=20.0)
    K, V = synth.kv_layer(31, 0, topics, G, d)
    off = oracle.segment(toks[0], synth.BOUNDARY_IDS, tau)
    Kf = synth.bf16_bits_to_f32(K).copy()
    for s, val in ((5, np.nan), (9, np.inf), (14, -np.inf), (20, np.nan), (33, np.inf)):
        Kf[0, 0, off[s], s % d] = val                       # one poisoned coordinate
    Kf[0, 0, off[40]:off[41]] = -0.0                         # a sentence of negative zeros
    Kf[0, 0, off[41]:off[42]] = 0.0                          # ... and one of positive zeros
    K = synth.f32_to_bf16_bits(Kf)
    dev = cuda_device
    skv = _skv(B, 1, Hq, G, d, L, tau)
    orc = oracle.Oracle(toks, synth.BOUNDARY_IDS, tau, 1, Hq, G, d)
    Kd, Vd = from_bits(K, dev), from_bits(V, dev)
    skv.prefill_compress(0, Kd, Vd, token_ids=torch.from_numpy(toks).to(dev), boundary_ids=synth.BOUNDARY_IDS)
    orc.prefill_layer(0, K, V)
    E = to_bits(skv.embeddings(0))
    S = skv.sentence_counts()[0]
    # bit-exact, except that a NaN's payload is not part of the canonical arithmetic (A7: NaN stays NaN)
    Eg, Eo = E[0, 0, :S], orc.E[0][0][0]
    nan_g, nan_o = np.isnan(synth.bf16_bits_to_f32(Eg)), np.isnan(synth.bf16_bits_to_f32(Eo))
    assert np.array_equal(nan_g, nan_o) and nan_o.any()
    assert np.array_equal(Eg[~nan_o], Eo[~nan_o])
    ids = torch.empty((B, G, tau), dtype=torch.int32, device=dev)
    out = torch.empty((B, Hq, d), dtype=torch.float32, device=dev)
    rng = np.random.default_rng(5)
    seen_nonfinite = False
    for s in range(steps):
        qf = rng.standard_normal((B, Hq, d)).astype(np.float32)
        if s == 2:
            qf[:] = 0.0  # q = 0: Inf * 0 = NaN scores for the infinite sentences
        q = synth.f32_to_bf16_bits(qf)
        it = torch.full((B,), 500, dtype=torch.int32, device=dev)
        if mode == "split":
            skv.decode_select(0, from_bits(q, dev), it, ids)
            skv.decode_attend(0, from_bits(q, dev), out)
        else:
            skv.decode_step(0, from_bits(q, dev), it, out, ids)
        sc_o, ids_o, _ = orc.decode_select(0, q, np.array([500]))
        O_o = orc.decode_attend(0, q, ids_o)
        sc_g = skv.scores(0).cpu().numpy()[0, 0, :S]
        so = sc_o[0][0]
        assert np.array_equal(np.isnan(sc_g), np.isnan(so)), f"NaN scores s={s}"
        assert np.array_equal(sc_g[~np.isnan(so)].view(np.uint32), so[~np.isnan(so)].view(np.uint32)), f"scores s={s}"
        seen_nonfinite |= not np.all(np.isfinite(sc_o[0][0]))
        n = len(ids_o[0][0])
        got = ids.cpu().numpy()
        assert np.array_equal(got[0, 0, :n], ids_o[0][0]) and np.all(got[0, 0, n:] == -1), f"ids s={s}"
        O_g = out.cpu().numpy()
        fin = np.isfinite(O_o) & np.isfinite(O_g)
        assert np.array_equal(np.isfinite(O_o), np.isfinite(O_g))
        assert np.all(np.abs(O_g[fin] - O_o[fin]) <= ATOL)
    assert seen_nonfinite
