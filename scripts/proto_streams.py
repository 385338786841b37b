#!/usr/bin/env python3
"""Prototype: per-layer fork/join of the batch's sequences over CUDA streams (one context per
sequence shard), so one sequence's latency-bound selection overlaps another's HBM-bound scoring /
attention.  Compares step time for nsplit in {1, 2, 4} at the 8b-128k device-resident shapes."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2504_00970_b200 as skvlib, synth

B, M, Hq, G, d, L, tau = 4, 32, 32, 8, 128, 131072, 2048
dev = torch.device("cuda:0")
toks, topics = synth.prompts(0, B, L, 25.0)
top = torch.from_numpy(topics).to(dev)
KV = [synth.kv_layer_torch(0, l, top, G, d, device=dev) for l in range(M)]
gen = torch.Generator(device=dev); gen.manual_seed(3)
tgt = torch.zeros(B, dtype=torch.int32, device=dev)
POOL = 4
qs = [[synth.queries_torch(gen, KV[l][2], tgt, Hq, G, d).contiguous() for l in range(M)] for _ in range(POOL)]
it = torch.full((B,), 300, dtype=torch.int32, device=dev)
res = {}
for nsplit in (1, 2, 4):
    bs = B // nsplit
    ctxs = [skvlib.SentenceKV(batch=B, layers=M, q_heads=Hq, kv_heads=G, head_dim=d, max_context=L, token_budget=tau,
                              batch_begin=i * bs, batch_count=bs) for i in range(nsplit)]
    for i, c in enumerate(ctxs):
        for l in range(M):
            c.prefill_compress(l, KV[l][0][i * bs:(i + 1) * bs].contiguous() if nsplit > 1 else KV[l][0],
                               KV[l][1][i * bs:(i + 1) * bs].contiguous() if nsplit > 1 else KV[l][1],
                               torch.from_numpy(toks[i * bs:(i + 1) * bs].copy()).to(dev) if l == 0 else None,
                               synth.BOUNDARY_IDS if l == 0 else None)
    torch.cuda.synchronize()
    qsl = [[[q[i * bs:(i + 1) * bs].contiguous() for q in qs[p]] for i in range(nsplit)] for p in range(POOL)]
    its = [it[i * bs:(i + 1) * bs].contiguous() for i in range(nsplit)]
    outs = [[torch.empty((bs, Hq, d), dtype=torch.float32, device=dev) for _ in range(M)] for _ in range(nsplit)]
    streams = [torch.cuda.Stream(device=dev) for _ in range(nsplit)]
    def step(p):
        main = torch.cuda.current_stream()
        for l in range(M):
            ev = torch.cuda.Event()
            ev.record(main)
            for i in range(nsplit):
                streams[i].wait_event(ev)
                with torch.cuda.stream(streams[i]):
                    ctxs[i].decode_step(l, qsl[p][i][l], its[i], outs[i][l])
            for i in range(nsplit):
                e2 = torch.cuda.Event()
                e2.record(streams[i])
                main.wait_event(e2)
    for p in range(POOL):
        step(p)
    torch.cuda.synchronize()
    cs = torch.cuda.Stream(device=dev)
    graphs = []
    with torch.cuda.stream(cs):
        for p in range(POOL):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cs):
                step(p)
            graphs.append(g)
    torch.cuda.synchronize()
    for w in range(10):
        graphs[w % POOL].replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 200
    e0.record()
    for k in range(K):
        graphs[k % POOL].replay()
    e1.record()
    torch.cuda.synchronize()
    res[nsplit] = e0.elapsed_time(e1) / K
    print(f"nsplit={nsplit}: {res[nsplit]:.4f} ms/step", flush=True)
    for c in ctxs:
        c.close()
