"""GPU parity of SURVEY 8(f) NEXT-2 (local segment + context growth, reading A29) against the oracle,
through the C ABI: each step appends the token's K/V (sentencekv_decode_append), completed generated
sentences become buckets (their embeddings bit-exact), scores and selected ids (including generated
sentences) bit-exact, O over selection + local segment within 2e-3."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests.gpu_harness import ATOL, from_bits, to_bits

pytestmark = pytest.mark.gpu


def _run(mode, seed=0, B=2, M=1, Hq=8, G=2, d=64, L=3000, tau=128, steps=40, mean_sentence=6.0, max_generated=64,
         graph=False, residency="device"):
    import paper_2504_00970_b200 as skvlib

    dev = torch.device("cuda:0")
    toks, topics = synth.prompts(seed, B, L, median=20.0)
    Ks, Vs = zip(*(synth.kv_layer(seed, l, topics, G, d) for l in range(M)))
    skv = skvlib.SentenceKV(batch=B, layers=M, q_heads=Hq, kv_heads=G, head_dim=d, max_context=L, token_budget=tau,
                            max_generated=max_generated,
                            residency=skvlib.SKV_KV_HOST if residency == "host" else skvlib.SKV_KV_DEVICE)
    orc = oracle.Oracle(toks, synth.BOUNDARY_IDS, tau, M, Hq, G, d, max_generated=max_generated)
    Kd = [from_bits(K, dev) for K in Ks]
    Vd = [from_bits(V, dev) for V in Vs]
    tok_dev = torch.from_numpy(toks).to(dev)
    for l in range(M):
        skv.prefill_compress(l, Kd[l], Vd[l], token_ids=tok_dev if l == 0 else None,
                             boundary_ids=synth.BOUNDARY_IDS if l == 0 else None)
        orc.prefill_layer(l, Ks[l], Vs[l])
    S0 = skv.sentence_counts()
    script, target = synth.decode_script(seed, B, steps, mean_sentence=mean_sentence)
    rng = np.random.default_rng(seed + 100)
    ids = torch.empty((B, G, tau), dtype=torch.int32, device=dev)
    out = torch.empty((B, Hq, d), dtype=torch.float32, device=dev)
    worst, grown = 0.0, 0
    for s in range(steps):
        it = torch.from_numpy(script[s]).to(dev)
        for l in range(M):
            kg = synth.f32_to_bf16_bits(rng.standard_normal((B, G, d)).astype(np.float32) + 0.5)
            vg = synth.f32_to_bf16_bits(rng.standard_normal((B, G, d)).astype(np.float32))
            q = synth.queries(seed, l, s, target[s], Hq, G, d)
            skv.decode_append(l, from_bits(kg, dev), from_bits(vg, dev), it)
            orc.decode_append(l, kg, vg, script[s])
            if mode == "split":
                skv.decode_select(l, from_bits(q, dev), it, ids)
                skv.decode_attend(l, from_bits(q, dev), out)
            else:
                skv.decode_step(l, from_bits(q, dev), it, out, ids)
            sc_o, ids_o, _ = orc.decode_select(l, q, script[s])
            O_o = orc.decode_attend(l, q, ids_o)
            sc_g = skv.scores(l).cpu().numpy()
            E = to_bits(skv.embeddings(l))
            got, O_g = ids.cpu().numpy(), out.cpu().numpy()
            for b in range(B):
                nb = len(orc.offsets(l, b)) - 1
                grown = max(grown, nb - S0[b])
                for g in range(G):
                    assert np.array_equal(E[b, g, S0[b]:nb], orc.E[l][b][g][S0[b]:nb]), f"generated E s={s} l={l}"
                    assert np.array_equal(sc_g[b, g, :nb].view(np.uint32), sc_o[b][g].view(np.uint32)), \
                        f"scores s={s} l={l} b={b} g={g}"
                    n = len(ids_o[b][g])
                    assert np.array_equal(got[b, g, :n], ids_o[b][g]) and np.all(got[b, g, n:] == -1), \
                        f"ids s={s} l={l} b={b} g={g}"
            err = float(np.abs(O_g - O_o).max())
            assert err <= ATOL, f"O s={s} l={l}: {err}"
            worst = max(worst, err)
    skv.sync()
    return worst, grown


@pytest.mark.parametrize("mode", ["split", "step"])
def test_local_segment_and_growth(cuda_device, mode):
    worst, grown = _run(mode)
    assert grown >= 3  # several generated sentences became buckets


@pytest.mark.parametrize("mode", ["split", "step"])
def test_local_segment_host_residency(cuda_device, mode):
    """The same with the prompt's K/V offloaded to pinned host memory (P3): context rows through the
    working set / page cache, generated rows (local segment and generated buckets) from HBM."""
    worst, grown = _run(mode, seed=4, residency="host")
    assert grown >= 3


def test_local_host_residency_d128_two_layers(cuda_device):
    _run("step", seed=5, B=1, M=2, Hq=16, G=4, d=128, L=2500, tau=64, steps=40, mean_sentence=12.0, residency="host")


@pytest.mark.parametrize("mode", ["split", "step"])
def test_local_d128_gqa4_two_layers_tau_cap(cuda_device, mode):
    """d = 128, grp = 4, 2 layers; tau = 40 with long generated sentences (mean 30): the A5 cap closes them."""
    _run(mode, seed=1, B=1, M=2, Hq=16, G=4, d=128, L=2500, tau=40, steps=50, mean_sentence=30.0)


def test_local_overflow_is_a_state_error(cuda_device):
    """More appends than max_generated: the token is dropped and sentencekv_sync reports STATE."""
    import paper_2504_00970_b200 as skvlib

    B, Hq, G, d, L = 1, 8, 2, 64, 1000
    toks, topics = synth.prompts(2, B, L, median=20.0)
    K, V = synth.kv_layer(2, 0, topics, G, d)
    skv = skvlib.SentenceKV(batch=B, layers=1, q_heads=Hq, kv_heads=G, head_dim=d, max_context=L, token_budget=64,
                            max_generated=4)
    Kd, Vd = from_bits(K, cuda_device), from_bits(V, cuda_device)
    skv.prefill_compress(0, Kd, Vd, token_ids=torch.from_numpy(toks).to(cuda_device), boundary_ids=synth.BOUNDARY_IDS)
    kv = torch.zeros((B, G, d), dtype=torch.bfloat16, device=cuda_device)
    it = torch.full((B,), 9, dtype=torch.int32, device=cuda_device)
    for _ in range(4):
        skv.decode_append(0, kv, kv, it)
    skv.sync()
    skv.decode_append(0, kv, kv, it)
    with pytest.raises(skvlib.SkvError, match="STATE"):
        skv.sync()


@pytest.mark.parametrize("mode", ["split", "step"])
def test_local_with_retention(cuda_device, mode):
    """NEXT-1 + NEXT-2 together (a serving loop with retention): the retained pool's buckets, the local
    segment -- the observation window, then the sentence being generated (always attended) -- and the
    completed generated sentences (buckets; sel_ids = the prompt's sentence count + k; the first one
    holds the window's rows too, reading A29)."""
    import paper_2504_00970_b200 as skvlib

    dev = cuda_device
    B, M, Hq, G, d, L, N, steps, seed = 1, 1, 32, 8, 128, 3000, 32, 30, 3
    toks, topics = synth.prompts(seed, B, L, median=20.0)
    Ks, Vs = zip(*(synth.kv_layer(seed, l, topics, G, d) for l in range(M)))
    # the window asks about 3 topics (as in test_gpu_retention): the retained set is unambiguous
    for k in range(100):
        pick = np.random.default_rng(seed * 1000 + k).choice(synth.N_TOPICS, 3, replace=False)
        count = int(np.isin(topics[0, :L - N], pick).sum())
        if count % 2 == 0:
            break
    tau = count // 2
    qw = [synth.window_queries(seed, l, pick[np.arange(N) % 3][None, :], Hq, G, d, scale=3.0) for l in range(M)]
    skv = skvlib.SentenceKV(batch=B, layers=M, q_heads=Hq, kv_heads=G, head_dim=d, max_context=L, token_budget=tau,
                            semantic_factor=2.0, obs_window=N, max_generated=64)
    orc = oracle.Oracle(toks, synth.BOUNDARY_IDS, tau, M, Hq, G, d, obs_window=N, semantic_factor=2.0,
                        max_generated=64)
    tok_dev = torch.from_numpy(toks).to(dev)
    for l in range(M):
        skv.prefill_compress(l, from_bits(Ks[l], dev), from_bits(Vs[l], dev), token_ids=tok_dev if l == 0 else None,
                             boundary_ids=synth.BOUNDARY_IDS if l == 0 else None, q_window=from_bits(qw[l], dev))
        orc.prefill_layer(l, Ks[l], Vs[l], q_window=qw[l])
    skv.sync()
    assert np.array_equal(skv.retained(0)[0].cpu().numpy()[0], orc.keep[0][0])
    script, target = synth.decode_script(seed, B, steps, mean_sentence=5.0)
    rng = np.random.default_rng(seed + 7)
    ids = torch.empty((B, G, tau), dtype=torch.int32, device=dev)
    out = torch.empty((B, Hq, d), dtype=torch.float32, device=dev)
    S_prompt = len(orc.off[0]) - 1
    n_pool = len(orc.sid[0][0])
    grown = False
    for s in range(steps):
        it = torch.from_numpy(script[s]).to(dev)
        for l in range(M):
            kg = synth.f32_to_bf16_bits(rng.standard_normal((B, G, d)).astype(np.float32) + 0.5)
            vg = synth.f32_to_bf16_bits(rng.standard_normal((B, G, d)).astype(np.float32))
            q = synth.queries(seed, l, s, target[s], Hq, G, d)
            skv.decode_append(l, from_bits(kg, dev), from_bits(vg, dev), it)
            orc.decode_append(l, kg, vg, script[s])
            if mode == "split":
                skv.decode_select(l, from_bits(q, dev), it, ids)
                skv.decode_attend(l, from_bits(q, dev), out)
            else:
                skv.decode_step(l, from_bits(q, dev), it, out, ids)
            _, ids_o, _ = orc.decode_select(l, q, script[s])
            O_o = orc.decode_attend(l, q, ids_o)
            got = ids.cpu().numpy()
            for g in range(G):
                want = orc.sid[l][0][ids_o[0][g]]
                grown |= bool(np.any(want >= S_prompt))
                n = len(want)
                assert np.array_equal(got[0, g, :n], want) and np.all(got[0, g, n:] == -1), f"ids s={s} g={g}"
            err = float(np.abs(out.cpu().numpy() - O_o).max())
            assert err <= ATOL, f"O s={s}: {err}"
            nb = len(orc.sid[l][0])  # generated buckets' E (the first includes the window's keys): bit-exact
            E = to_bits(skv.embeddings(l))
            for g in range(G):
                assert np.array_equal(E[0, g, n_pool:nb], orc.E[l][0][g][n_pool:nb]), f"generated E s={s} g={g}"
    skv.sync()
    gen = orc.sid[0][0][n_pool:]
    assert len(gen) >= 3 and np.array_equal(gen, S_prompt + np.arange(len(gen)))  # generated buckets appeared
