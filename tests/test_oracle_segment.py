"""Pins for the oracle's P1 segmentation -- CPU only."""
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden", "segmentation.txt")
PUNCT = {".": 1, "?": 2, "!": 3}
BSET = np.array(sorted(PUNCT.values()), dtype=np.int32)


def _golden():
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        wid, tau, toks, spans = (x.strip() for x in line.split("|"))
        vocab = {}
        ids = [PUNCT[w] if w in PUNCT else vocab.setdefault(w, 100 + len(vocab)) for w in toks.split()]
        want = [tuple(int(v) for v in sp.strip("[)").split(",")) for sp in spans.split()]
        yield wid, int(tau), np.array(ids, np.int32), want


@pytest.mark.parametrize("wid,tau,ids,want", list(_golden()))
def test_worked_strings(wid, tau, ids, want):
    off = oracle.segment(ids, BSET, tau if tau > 0 else len(ids) + 1)
    got = [(int(off[i]), int(off[i + 1])) for i in range(len(off) - 1)]
    assert got == want, wid


def _check_invariants(tokens, bset, tau, off):
    L = len(tokens)
    isb = np.isin(tokens, bset)
    # partition of [0, L) into non-empty spans
    assert off[0] == 0 and off[-1] == L
    assert np.all(np.diff(off) >= 1)
    assert np.all(np.diff(off) <= tau)  # reading A5: tau-cap
    for s in range(len(off) - 1):
        a, b = int(off[s]), int(off[s + 1])
        # no interior boundary token
        assert not isb[a : b - 1].any()
        # every span ends at a boundary, at L-1, or after exactly tau tokens
        assert isb[b - 1] or b == L or (b - a) == tau
    # closed-form count: the uncapped sentences have lengths T_i given by the boundary
    # positions (ends = boundary positions + the last token); the cap cuts each into
    # ceil(T_i / tau) pieces.
    ends = np.unique(np.concatenate([np.nonzero(isb)[0], [L - 1]]))
    T = np.diff(np.concatenate([[-1], ends]))
    assert len(off) - 1 == int(np.sum((T + tau - 1) // tau))


@pytest.mark.parametrize("seed", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("tau", [3, 17, 64, 256, 100000])
def test_invariants_on_synthetic_streams(seed, tau):
    toks, _ = synth.token_stream(seed, 0, 3000, median=20.0)
    off = oracle.segment(toks, synth.BOUNDARY_IDS, tau)
    _check_invariants(toks, synth.BOUNDARY_IDS, tau, off)


def test_no_boundaries_and_all_boundaries():
    L = 1000
    off = oracle.segment(np.full(L, 500, np.int32), BSET, 64)
    assert list(np.diff(off)) == [64] * (L // 64) + [L % 64]
    off = oracle.segment(np.full(L, 1, np.int32), BSET, 64)
    assert len(off) == L + 1 and np.all(np.diff(off) == 1)


def test_hundreds_of_sentences_at_32k():
    # "a 32K token input might be split into hundreds of sentence buckets"
    toks, _ = synth.token_stream(0, 0, 32768)
    S = len(oracle.segment(toks, synth.BOUNDARY_IDS, 1024)) - 1
    assert 100 <= S <= 3000
