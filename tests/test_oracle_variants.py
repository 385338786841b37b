"""Pins for the oracle's NEXT-3 paper variants and NEXT-4 Quest pages -- CPU only:
equal-size chunks (Sec. 6.1), outlier split, current-token query (Sec. 6.2),
skip-and-continue budget fill (alternative to reading A13), Quest page bounds (App. Quest)."""
import itertools

import numpy as np
import pytest

import oracle
import synth


def off_of(lengths):
    return np.concatenate([[0], np.cumsum(lengths)]).astype(np.int32)


# ----------------------------------------------------------------------------- equal chunks


@pytest.mark.parametrize("L,S,tau,want", [
    (10, 3, 256, [0, 4, 8, 10]),     # ceil(10/3) = 4
    (12, 3, 256, [0, 4, 8, 12]),
    (7, 7, 256, list(range(8))),     # one token each
    (100, 1, 30, [0, 30, 60, 90, 100]),  # one sentence: chunk length capped at tau (A5 / A26)
    (5, 9, 256, list(range(6))),     # more sentences than tokens cannot happen, but stays a partition
])
def test_equal_chunks_worked(L, S, tau, want):
    assert oracle.equal_chunks(L, S, tau).tolist() == want


@pytest.mark.parametrize("seed", range(4))
def test_equal_chunks_partition_and_count(seed):
    rng = np.random.default_rng(seed)
    L = int(rng.integers(1, 5000))
    S = int(rng.integers(1, L + 1))
    off = oracle.equal_chunks(L, S, 10 ** 6)
    n = np.diff(off)
    assert off[0] == 0 and off[-1] == L and np.all(n > 0)
    assert np.all(n[:-1] == n[0]) and n[-1] <= n[0]          # equal, the last shorter
    assert n[0] == -(-L // S) and len(n) == -(-L // n[0])     # ceil(L / S) tokens, ceil(L / len) chunks


# ----------------------------------------------------------------------------- outlier split


def test_outlier_threshold_worked():
    """Lengths 2, 2, 2, 10: mean 4, std sqrt(12) = 3.464; n = 1 -> T = floor(7.464) = 7; n = 2 -> 10."""
    off = off_of([2, 2, 2, 10])
    assert oracle.outlier_threshold(off, 1.0) == 7
    assert oracle.outlier_threshold(off, 2.0) == 10
    assert oracle.outlier_threshold(off_of([5, 5, 5]), 3.0) == 5     # std 0 -> mean


@pytest.mark.parametrize("seed", range(4))
def test_outlier_threshold_matches_numpy_statistics(seed):
    lens = synth.sentence_lengths(seed, 0, 3000)
    off = off_of(lens)
    for n in (0.5, 1.0, 2.5):
        want = int(np.floor(np.mean(lens) + n * np.std(lens)))  # population std
        got = oracle.outlier_threshold(off, n)
        assert abs(got - want) <= 1 and (got == want or abs(np.mean(lens) + n * np.std(lens) - round(np.mean(lens) + n * np.std(lens))) < 1e-9)


def test_outlier_split_driver():
    """The split cuts only the sentences longer than T, into pieces of T tokens (the last shorter)."""
    toks, _ = synth.prompts(3, 1, 4000, median=25.0)
    plain = oracle.Oracle(toks, synth.BOUNDARY_IDS, 4096, 1, 2, 1, 64)
    split = oracle.Oracle(toks, synth.BOUNDARY_IDS, 4096, 1, 2, 1, 64, outlier_n=1.0)
    T = oracle.outlier_threshold(plain.off[0], 1.0)
    n0, n1 = np.diff(plain.off[0]), np.diff(split.off[0])
    assert n1.max() <= T < n0.max()
    want = [x for n in n0 for x in ([T] * (n // T) + ([n % T] if n % T else []))]
    assert n1.tolist() == want


# ----------------------------------------------------------------------------- skip-and-continue


def test_select_skip_worked():
    """SURVEY's worked example S1: n = [4,3,5,2], scores [.5,.9,.9,.1], tau = 10: the prefix rule stops at
    s0 (12 > 10) and takes {1, 2}; skip-and-continue skips s0 and still takes s3 -> {1, 2, 3}, 10 tokens."""
    ids, n = oracle.select_skip(np.array([0.5, 0.9, 0.9, 0.1], np.float32), off_of([4, 3, 5, 2]), 10)
    assert ids.tolist() == [1, 2, 3] and n == 10


@pytest.mark.parametrize("seed", range(6))
def test_select_skip_brute_force(seed):
    """Characterisation, by enumeration of all 2^S subsets: the output is the unique set G with
    s in G  <=>  n_s + (tokens of G ranked above s) <= tau, for every s (ties -> lower index, NaN last)."""
    rng = np.random.default_rng(seed)
    S = int(rng.integers(1, 11))
    lens = rng.integers(1, 9, size=S)
    sc = (rng.integers(0, 4, size=S) / 2.0).astype(np.float32)
    tau = int(rng.integers(1, 30))
    order = sorted(range(S), key=lambda s: (-sc[s], s))
    rank = {s: i for i, s in enumerate(order)}
    sols = []
    for mask in range(1 << S):
        G = {s for s in range(S) if mask >> s & 1}
        if all((s in G) == (lens[s] + sum(lens[t] for t in G if rank[t] < rank[s]) <= tau) for s in range(S)):
            sols.append(sorted(G))
    assert len(sols) == 1
    ids, n = oracle.select_skip(sc, off_of(lens), tau)
    assert ids.tolist() == sols[0] and n == sum(lens[s] for s in sols[0]) <= tau


def test_select_skip_contains_prefix():
    """The prefix selection is always a subset of the skip-and-continue selection."""
    rng = np.random.default_rng(9)
    for _ in range(50):
        S = int(rng.integers(1, 60))
        lens = rng.integers(1, 40, size=S)
        sc = rng.standard_normal(S).astype(np.float32)
        tau = int(rng.integers(1, 300))
        a, _ = oracle.select(sc, off_of(lens), tau)
        b, _ = oracle.select_skip(sc, off_of(lens), tau)
        assert set(a) <= set(b)


# ----------------------------------------------------------------------------- current-token query


def test_current_query_ignores_history():
    """query_mode 1 ranks by q_t alone: two decode histories that end in the same q_t select the
    same sentences; with the mean query (Eq. 2) they do not."""
    B, Hq, G, d, L, tau = 1, 4, 2, 64, 1500, 100
    toks, topics = synth.prompts(2, B, L, median=20.0)
    K, V = synth.kv_layer(2, 0, topics, G, d)
    q_end = synth.queries(2, 0, 9, np.array([5]), Hq, G, d)
    hist = [synth.queries(2, 0, s, np.array([s % 7]), Hq, G, d) for s in range(3)]
    res = {}
    for mode in (0, 1):
        for h in (0, 1):
            o = oracle.Oracle(toks, synth.BOUNDARY_IDS, tau, 1, Hq, G, d, query_mode=mode)
            o.prefill_layer(0, K, V)
            for q in (hist if h else hist[:1]):
                o.decode_select(0, q, np.array([300]))
            _, ids, _ = o.decode_select(0, q_end, np.array([300]))
            res[mode, h] = [x.tolist() for x in ids[0]]
    assert res[1, 0] == res[1, 1] and res[0, 0] != res[0, 1]


# ----------------------------------------------------------------------------- Quest pages


def test_quest_meta_is_elementwise_min_max():
    rng = np.random.default_rng(0)
    K = synth.f32_to_bf16_bits(rng.standard_normal((37, 64)).astype(np.float32))
    mn, mx = oracle.quest_meta(K, 16)
    Kf = synth.bf16_bits_to_f32(K)
    for p in range(3):
        blk = Kf[16 * p:16 * (p + 1)]
        assert np.array_equal(synth.bf16_bits_to_f32(mn[p]), blk.min(axis=0))
        assert np.array_equal(synth.bf16_bits_to_f32(mx[p]), blk.max(axis=0))


def test_quest_score_worked():
    """d = 16 (two lanes), one head: q = (1, -1, 0...), min = (0, 0, ...), max = (2, 1, ...):
    max(0, 2) + max(-0, -1) = 2."""
    q = np.zeros((1, 16), np.float32)
    q[0, 0], q[0, 1] = 1.0, -1.0
    mn = np.zeros((1, 16), np.float32)
    mx = np.zeros((1, 16), np.float32)
    mx[0, 0], mx[0, 1] = 2.0, 1.0
    b = synth.f32_to_bf16_bits
    assert oracle.quest_score(b(q), b(mn), b(mx)).tolist() == [2.0]


@pytest.mark.parametrize("P", [1, 16, 32])
def test_quest_bound_upper_bounds_every_token(P):
    """For every token x of page p: sum_h q_h . k_x <= U(p) (Quest's bound; fp32 rounding slack), with
    equality when the page has a single token (P = 1) or all its keys are identical."""
    rng = np.random.default_rng(P)
    grp, d, L = 4, 64, 200
    q = synth.f32_to_bf16_bits(rng.standard_normal((grp, d)).astype(np.float32))
    K = synth.f32_to_bf16_bits(rng.standard_normal((L, d)).astype(np.float32))
    if P == 32:
        K[32:64] = K[40]  # one page of identical keys
    mn, mx = oracle.quest_meta(K, P)
    U = oracle.quest_score(q, mn, mx).astype(np.float64)
    qf = synth.bf16_bits_to_f32(q).astype(np.float64)
    s = (synth.bf16_bits_to_f32(K).astype(np.float64) @ qf.T).sum(axis=1)  # sum over heads, per token
    for x in range(L):
        assert s[x] <= U[x // P] + 1e-4 * (1 + abs(U[x // P]))
    if P == 1:
        np.testing.assert_allclose(U, s, rtol=1e-5, atol=1e-4)
    if P == 32:
        assert abs(U[1] - s[40]) <= 1e-4 * (1 + abs(s[40]))


def test_quest_driver_selects_whole_pages():
    """Quest mode: fixed pages of P tokens, tau = 5 pages' worth selects the 5 best-bounded pages."""
    B, Hq, G, d, L, P = 1, 4, 2, 64, 1000, 16
    toks, topics = synth.prompts(4, B, L, median=20.0)
    K, V = synth.kv_layer(4, 0, topics, G, d)
    o = oracle.Oracle(toks, synth.BOUNDARY_IDS, 5 * P, 1, Hq, G, d, bucket_mode=2, chunk_size=P)
    o.prefill_layer(0, K, V)
    assert o.off[0].tolist() == list(range(0, 1000, 16)) + [1000]
    q = synth.queries(4, 0, 0, np.array([3]), Hq, G, d)
    sc, ids, ntok = o.decode_select(0, q, np.array([300]))
    for g in range(G):
        want = sorted(sorted(range(len(sc[0][g])), key=lambda p: (-sc[0][g][p], p))[:5])
        assert ids[0][g].tolist() == want and ntok[0][g] == 5 * P
