"""GPU parity of SURVEY 8(f) NEXT-3 (paper variants) and NEXT-4 (Quest pages) against the oracle's
twins, through the C ABI: bucket offsets, embeddings / page bounds, scores and selected ids bit-exact,
O max-abs <= 2e-3 -- for the split calls and decode_step (the one-launch kernel for the sentence-bucket
variants; the split kernels for Quest and skip-and-continue)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests.gpu_harness import ATOL, from_bits, to_bits

pytestmark = pytest.mark.gpu


def _run(mode, seed=0, B=2, M=1, Hq=8, G=2, d=64, L=4096, tau=256, steps=12, residency=0, **kw):
    import paper_2504_00970_b200 as skvlib

    dev = torch.device("cuda:0")
    toks, topics = synth.prompts(seed, B, L, median=20.0)
    Ks, Vs = zip(*(synth.kv_layer(seed, l, topics, G, d) for l in range(M)))
    skv = skvlib.SentenceKV(batch=B, layers=M, q_heads=Hq, kv_heads=G, head_dim=d, max_context=L, token_budget=tau,
                            residency=residency, **kw)
    orc = oracle.Oracle(toks, synth.BOUNDARY_IDS, tau, M, Hq, G, d, **kw)
    tok_dev = torch.from_numpy(toks).to(dev)
    Kd = [from_bits(K, dev) for K in Ks]  # device residency borrows K/V: keep them alive
    Vd = [from_bits(V, dev) for V in Vs]
    for l in range(M):
        skv.prefill_compress(l, Kd[l], Vd[l], token_ids=tok_dev if l == 0 else None,
                             boundary_ids=synth.BOUNDARY_IDS if l == 0 else None)
        orc.prefill_layer(l, Ks[l], Vs[l])
    skv.sync()
    S = skv.sentence_counts()
    off = skv.offsets().cpu().numpy()
    quest = kw.get("bucket_mode", 0) == 2
    for b in range(B):
        assert S[b] == len(orc.off[b]) - 1 and np.array_equal(off[b, :S[b] + 1], orc.off[b]), f"buckets b={b}"
    for l in range(M):
        E = to_bits(skv.embeddings(l))
        for b in range(B):
            for g in range(G):
                if quest:
                    mn, mx = orc.E[l][b][g]
                    assert np.array_equal(E[b, g, :S[b], 0], mn) and np.array_equal(E[b, g, :S[b], 1], mx)
                else:
                    assert np.array_equal(E[b, g, :S[b]], orc.E[l][b][g]), f"E l={l} b={b} g={g}"
    script, target = synth.decode_script(seed, B, steps)
    ids = torch.empty((B, G, tau), dtype=torch.int32, device=dev)
    cnt = torch.empty((B, G), dtype=torch.int32, device=dev)
    ntk = torch.empty((B, G), dtype=torch.int32, device=dev)
    out = torch.empty((B, Hq, d), dtype=torch.float32, device=dev)
    worst = 0.0
    for s in range(steps):
        it = torch.from_numpy(script[s]).to(dev)
        for l in range(M):
            q = synth.queries(seed, l, s, target[s], Hq, G, d)
            if mode == "split":
                skv.decode_select(l, from_bits(q, dev), it, ids, cnt, ntk)
                skv.decode_attend(l, from_bits(q, dev), out)
            else:
                skv.decode_step(l, from_bits(q, dev), it, out, ids, cnt, ntk)
            sc_o, ids_o, ntok_o = orc.decode_select(l, q, script[s])
            O_o = orc.decode_attend(l, q, ids_o)
            sc_g = skv.scores(l).cpu().numpy()
            got, c_g, t_g, O_g = ids.cpu().numpy(), cnt.cpu().numpy(), ntk.cpu().numpy(), out.cpu().numpy()
            for b in range(B):
                for g in range(G):
                    assert np.array_equal(sc_g[b, g, :S[b]].view(np.uint32), sc_o[b][g].view(np.uint32)), \
                        f"scores s={s} l={l} b={b} g={g}"
                    n = len(ids_o[b][g])
                    assert c_g[b, g] == n and t_g[b, g] == ntok_o[b][g] <= tau
                    assert np.array_equal(got[b, g, :n], ids_o[b][g]) and np.all(got[b, g, n:] == -1), \
                        f"ids s={s} l={l} b={b} g={g}"
            err = float(np.abs(O_g - O_o).max())
            assert err <= ATOL, f"O s={s} l={l}: {err}"
            worst = max(worst, err)
    return worst


@pytest.mark.parametrize("mode", ["split", "step"])
def test_equal_chunks(cuda_device, mode):
    """NEXT-3 Sec. 6.1: as many equal chunks as sentences (A26)."""
    _run(mode, bucket_mode=1)


@pytest.mark.parametrize("mode", ["split", "step"])
@pytest.mark.parametrize("n", [0.5, 1.5])
def test_outlier_split(cuda_device, mode, n):
    """NEXT-3 P:765: sentences longer than mean + n*std cut into pieces of T tokens (A27)."""
    _run(mode, seed=1, outlier_n=n)


@pytest.mark.parametrize("mode", ["split", "step"])
def test_current_token_query(cuda_device, mode):
    """NEXT-3 Sec. 6.2: rank by q_t instead of the Eq. 2 mean (d = 128, grp = 4, 2 layers)."""
    _run(mode, seed=2, M=2, Hq=16, G=4, d=128, L=3000, tau=200, query_mode=1)


@pytest.mark.parametrize("mode", ["split", "step"])
def test_skip_and_continue(cuda_device, mode):
    """NEXT-3: walk the whole ranking, take every sentence that still fits."""
    _run(mode, seed=3, fill_mode=1)


@pytest.mark.parametrize("mode", ["split", "step"])
@pytest.mark.parametrize("P", [16, 32])
def test_quest_pages(cuda_device, mode, P):
    """NEXT-4 App. Quest: fixed pages of P tokens, min/max bounds of the current query (A28)."""
    _run(mode, seed=4, bucket_mode=2, chunk_size=P)


def test_quest_pages_d128_gqa8_host_residency(cuda_device):
    """Quest at d = 128, grp = 8, host residency (pages fetched from the pinned store like sentences)."""
    _run("step", seed=5, B=1, M=2, Hq=16, G=2, d=128, L=5000, tau=512, residency=1, bucket_mode=2, chunk_size=16)


def test_variants_combined_skip_current_query(cuda_device):
    _run("step", seed=6, query_mode=1, fill_mode=1, bucket_mode=1)
