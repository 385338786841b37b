"""Pins for the oracle's NEXT-1 importance-filtered retention: token importance alpha
(reading A21), global top-floor(r*tau) retention, the retained
sentence buckets (reading A25) and the Algorithm 1 driver with a window -- CPU only."""
import os

import numpy as np
import pytest
import torch

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden", "retention.txt")


def _rand_case(seed, N, Hq, G, L, d, scale=1.0):
    rng = np.random.default_rng(seed)
    qw = synth.f32_to_bf16_bits(scale * rng.standard_normal((N, Hq, d)).astype(np.float32))
    K = synth.f32_to_bf16_bits(rng.standard_normal((G, L, d)).astype(np.float32))
    return qw, K


# ----------------------------------------------------------------------------- alpha


@pytest.mark.parametrize("N,Hq,G,L,d", [(4, 4, 2, 37, 64), (1, 2, 2, 9, 64), (8, 8, 2, 70, 128), (3, 8, 1, 20, 64)])
def test_alpha_equals_torch_softmax(N, Hq, G, L, d):
    """A second, independent implementation with library routines (fp64 matmul, masked softmax):
    causal softmax of every window row over its prefix, mass on [0, L-N) summed over rows and heads."""
    qw, K = _rand_case(N * 100 + L, N, Hq, G, L, d)
    got = oracle.window_importance(qw, K)
    q = torch.from_numpy(synth.bf16_bits_to_f32(qw).astype(np.float64))          # [N][Hq][d]
    k = torch.from_numpy(synth.bf16_bits_to_f32(K).astype(np.float64))           # [G][L][d]
    k = k.repeat_interleave(Hq // G, dim=0)                                       # [Hq][L][d]
    z = torch.einsum("whd,hld->hwl", q, k) / np.sqrt(d)                           # [Hq][N][L]
    pos = torch.arange(L - N, L)[:, None]
    z = z.masked_fill(torch.arange(L)[None, :] > pos, float("-inf"))
    p = torch.softmax(z, dim=-1)
    want = p[:, :, : L - N].sum(dim=(0, 1)).numpy()
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("zero_q", [False, True])
def test_alpha_uniform_closed_form(zero_q):
    """Identical keys (or q = 0) make every softmax uniform over the prefix, so
    alpha_j = Hq * sum_w 1 / (L - N + w + 1) for every candidate j (closed form)."""
    N, Hq, G, L, d = 5, 4, 2, 41, 64
    rng = np.random.default_rng(3)
    if zero_q:
        qw = np.zeros((N, Hq, d), np.uint16)
        K = synth.f32_to_bf16_bits(rng.standard_normal((G, L, d)).astype(np.float32))
    else:
        qw = synth.f32_to_bf16_bits(rng.standard_normal((N, Hq, d)).astype(np.float32))
        row = synth.f32_to_bf16_bits(rng.standard_normal((G, 1, d)).astype(np.float32))
        K = np.repeat(row, L, axis=1)
    got = oracle.window_importance(qw, K)
    want = Hq * sum(1.0 / (L - N + w + 1) for w in range(N))
    np.testing.assert_allclose(got, np.full(L - N, want), rtol=1e-13)


def test_alpha_one_hot_key():
    """A window query aligned with one key far more than with any other puts (almost) all of its
    mass there: alpha of that key -> the number of (window row, head) pairs that see it."""
    N, Hq, G, L, d = 2, 2, 1, 12, 64
    K = np.zeros((G, L, d), np.float32)
    for j in range(L):
        K[0, j, j % d] = 1.0  # orthonormal keys
    qw = np.zeros((N, Hq, d), np.float32)
    qw[:, :, 5] = 64.0  # 64 / sqrt(64) = 8 nats: exp(8) vs 1 for the others
    got = oracle.window_importance(synth.f32_to_bf16_bits(qw), synth.f32_to_bf16_bits(K))
    e8 = np.exp(8.0)
    want5 = sum(Hq * e8 / (e8 + (L - N + w)) for w in range(N))  # prefix of L-N+w+1 keys, one hot
    assert abs(got[5] - want5) < 1e-12
    assert np.argmax(got) == 5 and got[5] > 0.99 * N * Hq


def test_alpha_mass_bound():
    """Each softmax row sums to one: sum_j alpha_j <= Hq * N, with the rest on window tokens."""
    qw, K = _rand_case(11, 6, 4, 2, 50, 64, scale=3.0)
    a = oracle.window_importance(qw, K)
    assert np.all(a >= 0) and a.sum() <= 4 * 6 + 1e-9


# ----------------------------------------------------------------------------- retention


def _golden():
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        rid, k, alpha, keep = (x.strip() for x in line.split("|"))
        yield rid, int(k), [float(v) for v in alpha.split()], [int(v) for v in keep.split()]


@pytest.mark.parametrize("rid,k,alpha,keep", list(_golden()))
def test_retain_worked(rid, k, alpha, keep):
    assert oracle.retain(np.array(alpha), k).tolist() == keep, rid


@pytest.mark.parametrize("seed", range(5))
def test_retain_brute_force(seed):
    """Top-k by (alpha desc, index asc) == the k indices every other index is worse than,
    found by counting how many indices rank above each one; heavy ties."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 40))
    a = rng.integers(0, 5, size=n).astype(np.float64) / 4.0
    for k in (0, 1, n // 2, n, n + 3):
        above = [sum(1 for j in range(n) if a[j] > a[i] or (a[j] == a[i] and j < i)) for i in range(n)]
        want = [i for i in range(n) if above[i] < k]
        assert oracle.retain(a, k).tolist() == want


def test_retained_count_paper_example():
    """'in a 32K context with tau = 1024 and r = 2, we might initially retain 2048 tokens'."""
    assert oracle.retained_count(2.0, 1024) == 2048
    a = np.random.default_rng(0).random(32768 - 32)
    assert len(oracle.retain(a, oracle.retained_count(2.0, 1024))) == 2048
    assert oracle.retained_count(2.5, 1000) == 2500 and oracle.retained_count(1.0, 7) == 7


def test_retained_buckets_worked():
    """Sentences [0,3) [3,5) [5,9) [9,10); kept tokens {1, 2, 6, 9}: sentence 1 keeps nothing and is
    dropped (A25); the pool offsets count retained tokens per surviving sentence."""
    off2, sid = oracle.retained_buckets(np.array([0, 3, 5, 9, 10]), np.array([1, 2, 6, 9]))
    assert off2.tolist() == [0, 2, 3, 4] and sid.tolist() == [0, 2, 3]
    off2, sid = oracle.retained_buckets(np.array([0, 3, 5]), np.array([], np.int32))
    assert off2.tolist() == [0] and sid.tolist() == []
    off2, sid = oracle.retained_buckets(np.array([0, 3, 5]), np.arange(5))
    assert off2.tolist() == [0, 3, 5] and sid.tolist() == [0, 1]


# ----------------------------------------------------------------------------- driver


def test_driver_retention_equals_full_when_everything_is_kept():
    """floor(r*tau) >= L - N keeps every candidate: the buckets are the prompt's sentences cut at the
    window; with a budget that fits them all, the decode attends every bucket plus the observation
    window (A25) -- i.e. full attention over the whole prompt (fp64 SDPA, a library routine)."""
    B, M, Hq, G, d, L, tau, N = 1, 1, 4, 2, 64, 300, 300, 8
    toks, topics = synth.prompts(5, B, L, median=20.0)
    K, V = synth.kv_layer(5, 0, topics, G, d)
    qw = synth.f32_to_bf16_bits(np.random.default_rng(1).standard_normal((B, N, Hq, d)).astype(np.float32))
    orc = oracle.Oracle(toks, synth.BOUNDARY_IDS, tau, M, Hq, G, d, obs_window=N, semantic_factor=1.0)
    orc.prefill_layer(0, K, V, q_window=qw)
    assert orc.keep[0][0].tolist() == list(range(L - N))
    off = orc.off[0]
    cut = off[off < L - N]
    want = np.concatenate([cut, [L - N]]) if cut[-1] != L - N else cut
    assert orc.loff[0][0].tolist() == want.tolist()
    q = synth.queries(5, 0, 0, np.zeros(B, np.int32), Hq, G, d)
    _, ids, ntok = orc.decode_select(0, q, np.array([300], np.int32))
    assert all(n == L - N for n in ntok[0])  # every retained token selected (r * tau = 300 >= L - N)
    O = orc.decode_attend(0, q, ids)
    qf = torch.from_numpy(synth.bf16_bits_to_f32(q[0]).astype(np.float64)).view(G, Hq // G, 1, d)
    kf = torch.from_numpy(synth.bf16_bits_to_f32(K[0]).astype(np.float64)).unsqueeze(1).expand(-1, Hq // G, -1, -1)
    vf = torch.from_numpy(synth.bf16_bits_to_f32(V[0]).astype(np.float64)).unsqueeze(1).expand(-1, Hq // G, -1, -1)
    ref = torch.nn.functional.scaled_dot_product_attention(qf, kf, vf).reshape(Hq, d).numpy()
    np.testing.assert_allclose(O[0], ref, rtol=0, atol=1e-10)


def test_driver_retention_budget():
    """The pool holds exactly floor(r*tau) tokens; every bucket's E is the mean of its retained keys;
    a selection never exceeds tau retained tokens."""
    B, M, Hq, G, d, L, tau, N = 2, 1, 4, 2, 64, 2000, 100, 16
    toks, topics = synth.prompts(6, B, L, median=20.0)
    K, V = synth.kv_layer(6, 0, topics, G, d)
    qw = synth.f32_to_bf16_bits(np.random.default_rng(2).standard_normal((B, N, Hq, d)).astype(np.float32))
    orc = oracle.Oracle(toks, synth.BOUNDARY_IDS, tau, M, Hq, G, d, obs_window=N, semantic_factor=2.5)
    orc.prefill_layer(0, K, V, q_window=qw)
    for b in range(B):
        keep = orc.keep[0][b]
        assert len(keep) == 250 and np.all(np.diff(keep) > 0) and keep[-1] < L - N
        off2, sid = orc.loff[0][b], orc.sid[0][b]
        assert off2[-1] == 250 and np.all(np.diff(off2) > 0)
        for i, s in enumerate(sid):  # every kept token of bucket i lies in sentence s
            toks_i = keep[off2[i]:off2[i + 1]]
            assert np.all((toks_i >= orc.off[b][s]) & (toks_i < orc.off[b][s + 1]))
        g = 1
        E = orc.E[0][b][g]
        Kf = synth.bf16_bits_to_f32(K[b, g])
        for i in range(len(sid)):
            m = Kf[keep[off2[i]:off2[i + 1]]].astype(np.float64).mean(axis=0)
            assert np.max(np.abs(synth.bf16_bits_to_f32(E[i]) - m)) <= np.abs(m).max() * 2 ** -8 + 1e-6
    q = synth.queries(6, 0, 0, np.zeros(B, np.int32), Hq, G, d)
    _, ids, ntok = orc.decode_select(0, q, np.array([1, 1], np.int32))
    assert all(n <= tau for row in ntok for n in row)
