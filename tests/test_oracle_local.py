"""Pins for the oracle's NEXT-2 local segment and context growth (reading A29) --
CPU only: with a budget covering everything the decode equals full attention over the prompt and every
generated token (a library routine); completed generated sentences become buckets at the next append
whose embedding is the mean of their keys (Eq. 1); no append leaves the plain path unchanged."""
import numpy as np
import torch

import oracle
import synth


def _gen_kv(rng, B, G, d):
    f = lambda: synth.f32_to_bf16_bits(rng.standard_normal((B, G, d)).astype(np.float32))
    return f(), f()


def _setup(B=1, Hq=4, G=2, d=64, L=300, tau=4096, seed=0, max_generated=64):
    toks, topics = synth.prompts(seed, B, L, median=20.0)
    K, V = synth.kv_layer(seed, 0, topics, G, d)
    o = oracle.Oracle(toks, synth.BOUNDARY_IDS, tau, 1, Hq, G, d, max_generated=max_generated)
    o.prefill_layer(0, K, V)
    return o, K, V


def test_full_budget_equals_full_attention_over_prompt_and_generated():
    B, Hq, G, d, L = 1, 4, 2, 64, 300
    o, K, V = _setup(B, Hq, G, d, L)
    rng = np.random.default_rng(1)
    script, target = synth.decode_script(1, B, 25, mean_sentence=5.0)
    gk, gv = [], []
    for s in range(25):
        k, v = _gen_kv(rng, B, G, d)
        gk.append(k)
        gv.append(v)
        o.decode_append(0, k, v, script[s])
        q = synth.queries(1, 0, s, target[s], Hq, G, d)
        _, ids, _ = o.decode_select(0, q, script[s])
        O = o.decode_attend(0, q, ids)
        Kall = np.concatenate([K[0], np.stack([x[0] for x in gk], axis=1)], axis=1)  # [G][L+s+1][d]
        Vall = np.concatenate([V[0], np.stack([x[0] for x in gv], axis=1)], axis=1)
        qf = torch.from_numpy(synth.bf16_bits_to_f32(q[0]).astype(np.float64)).view(G, Hq // G, 1, d)
        kf = torch.from_numpy(synth.bf16_bits_to_f32(Kall).astype(np.float64)).unsqueeze(1)
        vf = torch.from_numpy(synth.bf16_bits_to_f32(Vall).astype(np.float64)).unsqueeze(1)
        ref = torch.nn.functional.scaled_dot_product_attention(qf, kf.expand(-1, Hq // G, -1, -1),
                                                               vf.expand(-1, Hq // G, -1, -1))
        np.testing.assert_allclose(O[0], ref.reshape(Hq, d).numpy(), rtol=0, atol=1e-10)


def test_growth_bookkeeping_and_eq1():
    """Boundary inputs at steps 2 and 6: the sentences [0, 3) and [3, 7) of generated tokens become buckets
    at the appends of steps 3 and 7, with rows L + [0, 3) and L + [3, 7) and E = bf16(mean of keys)."""
    B, Hq, G, d, L = 1, 4, 2, 64, 300
    o, K, V = _setup(B, Hq, G, d, L)
    S0 = len(o.off[0]) - 1
    rng = np.random.default_rng(2)
    bnd = int(synth.BOUNDARY_IDS[0])
    toks = [7, 7, bnd, 7, 7, 7, bnd, 7, 7]
    keys = []
    for s, t in enumerate(toks):
        k, v = _gen_kv(rng, B, G, d)
        keys.append(k[0])
        o.decode_append(0, k, v, np.array([t], np.int32))
        nb = len(o.offsets(0, 0)) - 1 - S0
        assert nb == (0 if s < 3 else 1 if s < 7 else 2), s
    off = o.offsets(0, 0)
    assert off[S0:].tolist() == [L, L + 3, L + 7]
    for i, (a, e) in enumerate(((0, 3), (3, 7))):
        for g in range(G):
            m = synth.bf16_bits_to_f32(np.stack([keys[t][g] for t in range(a, e)])).astype(np.float64).mean(axis=0)
            got = synth.bf16_bits_to_f32(o.E[0][0][g][S0 + i]).astype(np.float64)
            assert np.max(np.abs(got - m)) <= np.abs(m).max() * 2 ** -8 + 1e-7


def test_tau_cap_closes_long_generated_sentences():
    """A generated sentence reaching tau tokens is closed like a capped prompt sentence (A5)."""
    B, Hq, G, d, L, tau = 1, 4, 2, 64, 300, 4
    o, K, V = _setup(B, Hq, G, d, L, tau=tau)
    S0 = len(o.off[0]) - 1
    rng = np.random.default_rng(3)
    for s in range(10):
        k, v = _gen_kv(rng, B, G, d)
        o.decode_append(0, k, v, np.array([9], np.int32))
    assert o.offsets(0, 0)[S0:].tolist() == [L, L + 4, L + 8]


def test_no_append_is_the_plain_path():
    B, Hq, G, d, L = 2, 4, 2, 64, 500
    toks, topics = synth.prompts(4, B, L, median=20.0)
    K, V = synth.kv_layer(4, 0, topics, G, d)
    a = oracle.Oracle(toks, synth.BOUNDARY_IDS, 64, 1, Hq, G, d)
    b = oracle.Oracle(toks, synth.BOUNDARY_IDS, 64, 1, Hq, G, d, max_generated=16)
    a.prefill_layer(0, K, V)
    b.prefill_layer(0, K, V)
    q = synth.queries(4, 0, 0, np.array([1, 2]), Hq, G, d)
    ra = a.decode_select(0, q, np.array([9, 9]))
    rb = b.decode_select(0, q, np.array([9, 9]))
    assert all(np.array_equal(x, y) for x, y in zip(ra[1][0] + ra[1][1], rb[1][0] + rb[1][1]))
    np.testing.assert_array_equal(a.decode_attend(0, q, ra[1]), b.decode_attend(0, q, rb[1]))


def test_with_retention_full_budget_equals_full_attention():
    """NEXT-1 + NEXT-2 (reading A29 with retention): floor(r*tau) >= L - N keeps every prompt token, and a
    budget above everything selects every bucket, so the decode -- retained buckets, the always-attended
    observation window, the completed generated sentences and the sentence being generated -- is full
    attention over the prompt and every generated token (fp64 SDPA, a library routine); the generated
    buckets are named S + k (S = the prompt's sentence count) and their E is the mean of their keys --
    the first one's includes the window's N keys (the local segment when decoding starts, A29)."""
    B, Hq, G, d, L, N, tau = 1, 4, 2, 64, 300, 8, 400
    toks, topics = synth.prompts(5, B, L, median=20.0)
    K, V = synth.kv_layer(5, 0, topics, G, d)
    qw = synth.f32_to_bf16_bits(np.random.default_rng(6).standard_normal((B, N, Hq, d)).astype(np.float32))
    o = oracle.Oracle(toks, synth.BOUNDARY_IDS, tau, 1, Hq, G, d, obs_window=N, semantic_factor=1.0,
                      max_generated=64)
    o.prefill_layer(0, K, V, q_window=qw)
    assert o.keep[0][0].tolist() == list(range(L - N))
    S = len(o.off[0]) - 1
    n_pool = len(o.sid[0][0])
    rng = np.random.default_rng(7)
    script, target = synth.decode_script(5, B, 25, mean_sentence=5.0)
    gk, gv = [], []
    for s in range(25):
        k, v = _gen_kv(rng, B, G, d)
        gk.append(k)
        gv.append(v)
        o.decode_append(0, k, v, script[s])
        q = synth.queries(5, 0, s, target[s], Hq, G, d)
        _, ids, _ = o.decode_select(0, q, script[s])
        O = o.decode_attend(0, q, ids)
        Kall = np.concatenate([K[0], np.stack([x[0] for x in gk], axis=1)], axis=1)  # [G][L+s+1][d]
        Vall = np.concatenate([V[0], np.stack([x[0] for x in gv], axis=1)], axis=1)
        qf = torch.from_numpy(synth.bf16_bits_to_f32(q[0]).astype(np.float64)).view(G, Hq // G, 1, d)
        kf = torch.from_numpy(synth.bf16_bits_to_f32(Kall).astype(np.float64)).unsqueeze(1)
        vf = torch.from_numpy(synth.bf16_bits_to_f32(Vall).astype(np.float64)).unsqueeze(1)
        ref = torch.nn.functional.scaled_dot_product_attention(qf, kf.expand(-1, Hq // G, -1, -1),
                                                               vf.expand(-1, Hq // G, -1, -1))
        np.testing.assert_allclose(O[0], ref.reshape(Hq, d).numpy(), rtol=0, atol=1e-10)
    gen = o.sid[0][0][n_pool:]
    assert len(gen) >= 3 and gen.tolist() == list(range(S, S + len(gen)))
    starts = np.flatnonzero(np.isin(np.concatenate(script[:, 0:1]), synth.BOUNDARY_IDS)) + 1  # sentence ends
    first = np.concatenate([[0], starts[:len(gen) - 1]])
    for i in range(len(gen)):  # bucket n_pool + i = generated tokens [first_i, first_{i+1})
        a, e = int(first[i]), int(starts[i])
        for g in range(G):
            rows = [gk[t][0][g] for t in range(a, e)]
            if i == 0:
                rows = list(K[0][g][L - N:]) + rows
            m = synth.bf16_bits_to_f32(np.stack(rows)).astype(np.float64).mean(axis=0)
            got = synth.bf16_bits_to_f32(o.E[0][0][g][n_pool + i]).astype(np.float64)
            assert np.max(np.abs(got - m)) <= np.abs(m).max() * 2 ** -8 + 1e-7
