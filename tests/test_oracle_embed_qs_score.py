"""Pins for the oracle's P2 (Eq. 1), D1 (Eq. 2 + similarity) steps -- CPU only.

Eq. 1 mean keys: PAPER.md P:402-405.  Eq. 2 mean query: P:431-435.  Similarity q^T k: P:440-442.
"""
import numpy as np
import pytest

import oracle
import synth


def bits(x):
    return synth.f32_to_bf16_bits(np.asarray(x, np.float32))


def f32(h):
    return synth.bf16_bits_to_f32(h)


# ----------------------------------------------------------------------------- Eq. 1


def test_embed_worked_example():
    # keys (1,2) and (3,4) in one sentence -> mean (2,3)
    K = bits([[1, 2], [3, 4]])
    E = oracle.embed(np.pad(K, ((0, 0), (0, 0))), np.array([0, 2], np.int32))
    assert f32(E).tolist() == [[2.0, 3.0]]


def test_embed_singleton_is_the_key():
    rng = np.random.default_rng(0)
    K = bits(rng.standard_normal((50, 64)) * 3)
    off = np.arange(51, dtype=np.int32)  # 50 one-token sentences
    assert np.array_equal(oracle.embed(K, off), K)


@pytest.mark.parametrize("n", [1, 2, 7, 255, 4096])
def test_embed_identical_keys_exact(n):
    # n <= 2^16 identical bf16 keys: every partial sum j*k is exact in fp32 (8+16 bits), and
    # (n*k)/n = k exactly, so E == k bit for bit.
    rng = np.random.default_rng(n)
    k = bits(rng.standard_normal(128) * 5)
    K = np.tile(k, (n, 1))
    E = oracle.embed(K, np.array([0, n], np.int32))
    assert np.array_equal(E[0], k)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_embed_matches_fp64_mean_within_bound(seed):
    toks, topics = synth.prompts(seed, 1, 4096, median=20.0)
    off = oracle.segment(toks[0], synth.BOUNDARY_IDS, 256)
    K, _ = synth.kv_layer(seed, 0, topics, 1, 128)
    E = f32(oracle.embed(K[0, 0], off)).astype(np.float64)
    Kf = f32(K[0, 0]).astype(np.float64)
    for s in range(len(off) - 1):
        a, b = off[s], off[s + 1]
        mean = Kf[a:b].mean(axis=0)
        n = b - a
        # 1/2 ulp of bf16 (2^-8 relative) + fp32 accumulation error n * 2^-24 * max|k|
        bound = np.abs(mean) * 2.0**-8 + n * 2.0**-24 * np.abs(Kf[a:b]).max() * 2 + 1e-30
        assert np.all(np.abs(E[s] - mean) <= bound), s


# ----------------------------------------------------------------------------- Eq. 2


def test_mean_query_singleton_and_cancellation():
    rng = np.random.default_rng(1)
    q = bits(rng.standard_normal((4, 64)))
    Sq = np.zeros((4, 64), np.float32)
    cnt = np.zeros(1, np.int32)
    qbar = oracle.qs_append_mean(Sq, cnt, q)
    assert np.array_equal(qbar, f32(q)) and cnt[0] == 1
    neg = q ^ np.uint16(0x8000)  # -q (sign flip in bf16)
    qbar = oracle.qs_append_mean(Sq, cnt, neg)
    assert np.all(qbar == 0.0) and cnt[0] == 2
    oracle.qs_reset(Sq, cnt)
    assert cnt[0] == 0 and np.all(Sq == 0)


def test_mean_query_matches_fp64_mean():
    rng = np.random.default_rng(2)
    qs = [bits(rng.standard_normal((8, 128))) for _ in range(40)]
    Sq = np.zeros((8, 128), np.float32)
    cnt = np.zeros(1, np.int32)
    for i, q in enumerate(qs):
        qbar = oracle.qs_append_mean(Sq, cnt, q)
        ref = np.mean([f32(x).astype(np.float64) for x in qs[: i + 1]], axis=0)
        assert np.max(np.abs(qbar - ref)) <= (i + 1) * 2.0**-23 * 8 + 1e-6


def test_group_query_sums_heads_of_group():
    rng = np.random.default_rng(3)
    qbar = rng.standard_normal((8, 64)).astype(np.float32)
    for g in range(2):
        qt = oracle.group_query(qbar, 4, g)
        ref = qbar[4 * g : 4 * g + 4].astype(np.float64).sum(axis=0)
        assert np.max(np.abs(qt - ref)) <= 4 * 2.0**-23 * np.abs(qbar).max() * 4
    assert np.array_equal(oracle.group_query(qbar, 1, 5), qbar[5])


# ------------------------------------------------------------------------ similarity


@pytest.mark.parametrize("d", [64, 128])
def test_score_matches_fp64_dot_within_bound(d):
    rng = np.random.default_rng(d)
    E = bits(rng.standard_normal((300, d)) * 2)
    qt = (rng.standard_normal(d) * 4).astype(np.float32)
    sc = oracle.score(qt, E)
    Ef = f32(E).astype(np.float64)
    ref = Ef @ qt.astype(np.float64)
    bound = d * 2.0**-23 * (np.abs(Ef) @ np.abs(qt).astype(np.float64))
    assert np.all(np.abs(sc - ref) <= bound)


def test_score_one_hot_query_reads_one_coordinate():
    rng = np.random.default_rng(4)
    E = bits(rng.standard_normal((20, 128)))
    for j in (0, 7, 8, 127):
        qt = np.zeros(128, np.float32)
        qt[j] = 1.0
        assert np.array_equal(oracle.score(qt, E), f32(E)[:, j])


def test_score_zero_query_gives_positive_zero_or_zero():
    E = bits(np.random.default_rng(5).standard_normal((10, 64)))
    assert np.all(oracle.score(np.zeros(64, np.float32), E) == 0.0)
