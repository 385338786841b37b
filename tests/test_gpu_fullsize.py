"""Full-size parity at BASELINE.json configs[2] (Llama-3.1-8B shapes, 128K context, tau=2048, batch 4,
K/V offloaded to pinned host) in the launch configuration bench.py times (sentencekv_decode_step),
and at one rank's shard of configs[3] (256K context, tau=4096, heads 4..7 of 8, as rank 1 of a
2-GPU head split) and configs[4] (Llama-3.1-70B shapes: 64 query heads, grp 8; sequences 6..7 of
16, as one rank of an 8-GPU batch split): every sequence's segmentation is compared in full;
embeddings, scores, selections and attention outputs on a seeded sample of (b, g) units that the
oracle computes one by one."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests.gpu_harness import ATOL, to_bits

pytestmark = pytest.mark.gpu


def _fullsize(dev, residency, B, Hq, G, d, L, tau, units, steps=3, layer=1, b0=0, g0=0, Gl=None, graph=False):
    """One rank's shard: global sequences b0 .. b0+B-1, KV heads g0 .. g0+Gl-1 of G (query heads
    grp*g0 .. grp*(g0+Gl)-1).  units are shard-local (b, g).  graph: steps after the first run as
    bench.py runs them, one captured CUDA graph of both layers replayed with each step's inputs."""
    import paper_2504_00970_b200 as skvlib

    Gl = Gl or G - g0
    grp = Hq // G
    Hl = Gl * grp
    toks, topics = (np.stack(x) for x in zip(*(synth.token_stream(0, b, L, 25.0) for b in range(b0, b0 + B))))
    skv = skvlib.SentenceKV(batch=b0 + B, layers=2, q_heads=Hq, kv_heads=G, head_dim=d, max_context=L,
                            token_budget=tau,
                            residency=skvlib.SKV_KV_HOST if residency == "host" else skvlib.SKV_KV_DEVICE,
                            kv_head_begin=g0, kv_head_count=Gl, batch_begin=b0, batch_count=B)
    top = torch.from_numpy(topics).to(dev)
    KV = [synth.kv_layer_torch(0, l, top, G, d, device=dev, b_begin=b0, g_begin=g0, g_count=Gl) for l in range(2)]
    for l in range(2):
        skv.prefill_compress(l, KV[l][0], KV[l][1], torch.from_numpy(toks).to(dev) if l == 0 else None,
                             synth.BOUNDARY_IDS if l == 0 else None)
    skv.sync()
    Kh = {u: to_bits(KV[layer][0][u[0], u[1]]) for u in units}
    Vh = {u: to_bits(KV[layer][1][u[0], u[1]]) for u in units}

    # P1: every prompt of the shard, bit-exact
    S = skv.sentence_counts()
    offs = skv.offsets().cpu().numpy()
    off_o = [oracle.segment(toks[b], synth.BOUNDARY_IDS, tau) for b in range(B)]
    for b in range(B):
        assert np.array_equal(offs[b, : S[b] + 1], off_o[b])
    # P2: sampled units, bit-exact
    E = to_bits(skv.embeddings(layer))
    E_o = {u: oracle.embed(Kh[u], off_o[u[0]]) for u in units}
    for (b, g) in units:
        assert np.array_equal(E[b, g, : S[b]], E_o[(b, g)])

    gen = torch.Generator(device=dev)
    gen.manual_seed(7)
    script, target = synth.decode_script(0, b0 + B, steps)
    script, target = script[:, b0:].copy(), target[:, b0:].copy()
    h0 = g0 * grp
    Sq = np.zeros((B, Hl, d), np.float32)
    cnt = np.zeros((B, 1), np.int32)
    ids = torch.empty((B, Gl, tau), dtype=torch.int32, device=dev)
    out = torch.empty((B, Hl, d), dtype=torch.float32, device=dev)
    bset = set(synth.BOUNDARY_IDS.tolist())
    g_q0, g_q, g_it, g_o0 = (torch.empty_like(out, dtype=torch.bfloat16), torch.empty_like(out, dtype=torch.bfloat16),
                             torch.empty((B,), dtype=torch.int32, device=dev), torch.empty_like(out))
    cg = None
    for s in range(steps):
        tg = torch.from_numpy(target[s]).to(dev)
        q0 = synth.queries_torch(gen, KV[0][2], tg, Hq, G, d)[:, h0:h0 + Hl].contiguous()
        q = synth.queries_torch(gen, KV[layer][2], tg, Hq, G, d)[:, h0:h0 + Hl].contiguous()
        it = torch.from_numpy(script[s]).to(dev)
        if graph and s > 0:
            g_q0.copy_(q0)
            g_q.copy_(q)
            g_it.copy_(it)
            if cg is None:
                torch.cuda.synchronize()
                cs = torch.cuda.Stream(device=dev)
                with torch.cuda.stream(cs):
                    cg = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(cg, stream=cs):
                        skv.decode_step(0, g_q0, g_it, g_o0)
                        skv.decode_step(layer, g_q, g_it, out, sel_ids=ids)
                torch.cuda.synchronize()
            cg.replay()
            torch.cuda.synchronize()
        else:
            skv.decode_step(0, q0, it, torch.empty_like(out))  # layer 0 runs too, as in a real step
            skv.decode_step(layer, q, it, out, sel_ids=ids)
        qb = to_bits(q)
        sc = skv.scores(layer).cpu().numpy()
        got_ids = ids.cpu().numpy()
        O = out.cpu().numpy()
        for b in sorted({u[0] for u in units}):
            qbar = oracle.qs_append_mean(Sq[b], cnt[b], qb[b])
            for g in [u[1] for u in units if u[0] == b]:
                qt = oracle.group_query(qbar, grp, g)
                sc_o = oracle.score(qt, E_o[(b, g)])
                assert np.array_equal(sc[b, g, : S[b]].view(np.uint32), sc_o.view(np.uint32)), (s, b, g)
                sel, _ = oracle.select(sc_o, off_o[b], tau)
                assert np.array_equal(got_ids[b, g, : len(sel)], sel) and np.all(got_ids[b, g, len(sel):] == -1)
                O_o = oracle.attend(qb[b, g * grp:(g + 1) * grp], Kh[(b, g)], Vh[(b, g)], off_o[b], sel)
                assert np.max(np.abs(O[b, g * grp:(g + 1) * grp] - O_o)) <= ATOL, (s, b, g)
            if int(script[s, b]) in bset:
                oracle.qs_reset(Sq[b], cnt[b])


@pytest.mark.parametrize("residency", ["host", "device"])
def test_config2_sampled_units(cuda_device, residency):
    """configs[2]: 8B shapes, 128K, tau 2048, batch 4, all heads (the bench's N=1 workload), in the
    bench's launch configuration (CUDA-graph replay after the first step)."""
    _fullsize(cuda_device, residency, B=4, Hq=32, G=8, d=128, L=131072, tau=2048,
              units=[(0, 0), (1, 3), (2, 5), (3, 7)], steps=4, graph=True)


def test_config3_head_shard_sampled_units(cuda_device):
    """configs[3]: 8B shapes, 256K context, tau 4096, batch 1; the shard of rank 1 of a 2-GPU head
    split (KV heads 4..7)."""
    _fullsize(cuda_device, "device", B=1, Hq=32, G=8, d=128, L=262144, tau=4096, units=[(0, 0), (0, 3)],
              g0=4, Gl=4)


def test_config4_70b_batch_shard_sampled_units(cuda_device):
    """configs[4]: 70B shapes (64 query heads, grp 8), 128K, tau 2048; the shard of one rank of an
    8-GPU batch split (sequences 6, 7 of 16, all 8 KV heads)."""
    _fullsize(cuda_device, "device", B=2, Hq=64, G=8, d=128, L=131072, tau=2048, units=[(0, 2), (1, 6)],
              b0=6)
