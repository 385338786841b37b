"""the per-layer all-gather of the per-head outputs fused into the attention epilogue
(sentencekv_set_output_peers / sentencekv_wait_outputs).  Two "ranks" = two head-shard contexts on ONE
GPU, each on its own stream (as on two GPUs): every rank's kernels store their outputs into every
rank's rank-major gather buffer and count arrivals; after the wait both buffers hold the same
[world][B][Hq_loc][d] result, equal to the unsharded decode after parallel.assemble.  The NVLink
transport itself needs two GPUs (not available in this round); the kernel path, the layout and the
flag protocol are the same."""
import numpy as np
import pytest
import torch

import synth
from paper_2504_00970_b200 import parallel
from tests.gpu_harness import from_bits

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", ["step", "split"])
def test_fused_gather_two_head_shards_one_gpu(cuda_device, mode):
    import paper_2504_00970_b200 as skvlib

    dev = cuda_device
    B, M, Hq, G, d, L, tau, world, steps = 2, 2, 16, 4, 128, 3000, 200, 2, 5
    toks, topics = synth.prompts(7, B, L, median=20.0)
    Ks = [from_bits(synth.kv_layer(7, l, topics, G, d)[0], dev) for l in range(M)]
    Vs = [from_bits(synth.kv_layer(7, l, topics, G, d)[1], dev) for l in range(M)]
    plans = [parallel.plan(B, G, Hq, world, r, "heads") for r in range(world)]
    ctxs = [skvlib.SentenceKV(layers=M, head_dim=d, max_context=L, token_budget=tau, **p.ctx_kwargs()) for p in plans]
    full = skvlib.SentenceKV(batch=B, layers=M, q_heads=Hq, kv_heads=G, head_dim=d, max_context=L, token_budget=tau)
    tok = torch.from_numpy(toks).to(dev)
    keep = []  # device residency borrows K/V: the shard copies must outlive the decode
    for l in range(M):
        for r, (p, c) in enumerate(zip(plans, ctxs)):
            g0, gn = p.kv_head_begin, p.kv_head_count
            keep.append((Ks[l][:, g0:g0 + gn].contiguous(), Vs[l][:, g0:g0 + gn].contiguous()))
            c.prefill_compress(l, keep[-1][0], keep[-1][1],
                               token_ids=tok if l == 0 else None, boundary_ids=synth.BOUNDARY_IDS if l == 0 else None)
        full.prefill_compress(l, Ks[l], Vs[l], token_ids=tok if l == 0 else None,
                              boundary_ids=synth.BOUNDARY_IDS if l == 0 else None)
    Hl = plans[0].q_head_count
    bufs = [[torch.full((world, B, Hl, d), float("nan"), device=dev) for _ in range(world)] for _ in range(M)]
    flags = [torch.zeros(world, dtype=torch.int32, device=dev) for _ in range(M)]
    for l in range(M):
        for r, c in enumerate(ctxs):
            c.set_output_peers(l, r, bufs[l], [flags[l].data_ptr() + 4 * p for p in range(world)])
    streams = [torch.cuda.Stream(device=dev) for _ in range(world)]
    script, target = synth.decode_script(7, B, steps)
    out_full = torch.empty((B, Hq, d), dtype=torch.float32, device=dev)
    outs = [torch.empty((B, Hl, d), dtype=torch.float32, device=dev) for _ in range(world)]
    for s in range(steps):
        it = torch.from_numpy(script[s]).to(dev)
        for l in range(M):
            q = from_bits(synth.queries(7, l, s, target[s], Hq, G, d), dev)
            torch.cuda.synchronize()
            for r, (p, c) in enumerate(zip(plans, ctxs)):
                qr = q[:, p.q_head_begin:p.q_head_begin + Hl].contiguous()
                with torch.cuda.stream(streams[r]):
                    if mode == "step":
                        c.decode_step(l, qr, it, outs[r], stream=streams[r])
                    else:
                        c.decode_select(l, qr, it, stream=streams[r])
                        c.decode_attend(l, qr, outs[r], stream=streams[r])
                    c.wait_outputs(l, stream=streams[r])
            full.decode_step(l, q, it, out_full)
            torch.cuda.synchronize()
            for r in range(world):
                got = parallel.assemble(bufs[l][r], plans[r])
                assert torch.equal(bufs[l][r][r], outs[r]), "own slot"
                assert torch.allclose(got, out_full, atol=2e-3, rtol=0), f"s={s} l={l} rank {r}"
                assert torch.equal(bufs[l][0], bufs[l][1])
            assert int(flags[l][0]) == int(flags[l][1]) == (s + 1) * world * B * plans[0].kv_head_count
