#!/usr/bin/env python3
"""Phase timestamps (clock64 of block 0 / thread 0) of the decode kernels, from the SKV_TRACE
build (libsentencekv_trace.so).  Runs the 8b-128k shapes on 2 layers, a few decode steps."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["SKV_LIB"] = os.path.join(ROOT, "paper_2504_00970_b200", "libsentencekv_trace.so")
import numpy as np, torch
import paper_2504_00970_b200 as skvlib, synth

B, M, Hq, G, d, L, tau = 4, 2, 32, 8, 128, 131072, 2048
dev = torch.device("cuda:0")
toks, topics = synth.prompts(0, B, L, 25.0)
skv = skvlib.SentenceKV(batch=B, layers=M, q_heads=Hq, kv_heads=G, head_dim=d, max_context=L, token_budget=tau)
top = torch.from_numpy(topics).to(dev)
KV = [synth.kv_layer_torch(0, l, top, G, d, device=dev) for l in range(M)]
for l in range(M):
    skv.prefill_compress(l, KV[l][0], KV[l][1], torch.from_numpy(toks).to(dev) if l == 0 else None,
                         synth.BOUNDARY_IDS if l == 0 else None)
gen = torch.Generator(device=dev); gen.manual_seed(1)
tgt = torch.zeros(B, dtype=torch.int32, device=dev)
out = torch.empty((B, Hq, d), dtype=torch.float32, device=dev)
it = torch.full((B,), 300, dtype=torch.int32, device=dev)
lib = skvlib.lib
buf = (ctypes.c_longlong * 32)()
def rd(name):
    getattr(lib, f"sentencekv_debug_trace_{name}")(buf)
    return list(buf)
for step in range(4):
    for l in range(M):
        q = synth.queries_torch(gen, KV[l][2], tgt, Hq, G, d)
        skv.decode_select(l, q, it)
        torch.cuda.synchronize()
        sel = rd("select")

        att = [0] * 32
        skv.decode_step(l, q, it, out)
        torch.cuda.synchronize()
        mma = rd("mma")
    ghz = 1.965
    def show(name, t, slots):
        t0 = t[slots[0]]
        print(name, " ".join(f"{s}:{(t[s]-t0)/ghz/1e3:.2f}" for s in slots if t[s] >= t0 and t[s] - t0 < 1e9))
    print(f"--- step {step} (us since first stamp)")
    show("score ", sel, [24, 25, 26])
    show("select", sel, [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 20, 21, 22])

    show("mma   ", mma, list(range(0, 13)))
