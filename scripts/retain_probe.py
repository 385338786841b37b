#!/usr/bin/env python3
"""NEXT-1 retention: alpha error vs the fp64 oracle at test sizes, and the prefill time at full size."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import oracle, synth
import paper_2504_00970_b200 as skvlib
from tests.gpu_harness import from_bits

dev = torch.device("cuda:0")
FULL_ONLY = "full" in sys.argv[1:]
for (B, Hq, G, d, L, N, tau, scale) in [(2, 32, 8, 128, 2777, 32, 300, 1.0), (1, 8, 2, 64, 4096, 16, 256, 1.0),
                                          (1, 16, 2, 128, 3000, 32, 300, 2.0)][:0 if FULL_ONLY else 3]:
    toks, topics = synth.prompts(1, B, L, 20.0)
    K, V = synth.kv_layer(1, 0, topics, G, d)
    qw = synth.window_queries(1, 0, topics[:, L - N:], Hq, G, d, scale=scale)
    skv = skvlib.SentenceKV(batch=B, layers=1, q_heads=Hq, kv_heads=G, head_dim=d, max_context=L, token_budget=tau, obs_window=N)
    skv.prefill_compress(0, from_bits(K, dev), from_bits(V, dev), torch.from_numpy(toks).to(dev), synth.BOUNDARY_IDS, q_window=from_bits(qw, dev))
    skv.sync()
    a = skv.importance(0, L).cpu().numpy().astype(np.float64)
    keep = skv.retained(0)[0].cpu().numpy()
    for b in range(B):
        ar = oracle.window_importance(qw[b], K[b])
        rel = np.abs(a[b] - ar) / np.maximum(ar, 1e-30)
        kr = oracle.retain(ar, len(keep[b]))
        srt = np.sort(ar)[::-1]
        m = len(keep[b])
        print(f"B={B} Hq={Hq} G={G} d={d} L={L} N={N}: alpha max rel err {rel.max():.3g} (median {np.median(rel):.3g}), "
              f"sum {a[b].sum():.4f} vs {ar.sum():.4f}; keep equal {np.array_equal(kr, keep[b])}, "
              f"differ {len(set(kr) ^ set(keep[b]))}; gap at cut {(srt[m-1]-srt[m])/srt[m-1]:.3g}")
# full size: prefill time with retention, configs[2] shapes
B, Hq, G, d, L, N, tau = 4, 32, 8, 128, 131072, 32, 2048
toks, topics = synth.prompts(0, B, L, 25.0)
top = torch.from_numpy(topics).to(dev)
skv = skvlib.SentenceKV(batch=B, layers=2, q_heads=Hq, kv_heads=G, head_dim=d, max_context=L, token_budget=tau, obs_window=N)
skv2 = skvlib.SentenceKV(batch=B, layers=2, q_heads=Hq, kv_heads=G, head_dim=d, max_context=L, token_budget=tau)
gen = torch.Generator(device=dev); gen.manual_seed(3)
for l in range(2):
    K, V, c = synth.kv_layer_torch(0, l, top, G, d, device=dev)
    qw = synth.window_queries_torch(gen, c, top[:, L - N:], Hq, G, d).contiguous()
    for rep in range(3):
        for s, kw in ((skv, dict(q_window=qw)), (skv2, {})):
            s.set_profiling(True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            s.prefill_compress(l, K, V, torch.from_numpy(toks).to(dev) if l == 0 else None, synth.BOUNDARY_IDS if l == 0 else None, **kw)
            torch.cuda.synchronize()
            p = s.profile_read()
            s.set_profiling(False)
            if rep == 2:
                print(("retention " if kw else "plain     ") + f"layer {l}: wall {1e3*(time.perf_counter()-t0):.2f} ms; " +
                      ", ".join(f"{k}={v[0]:.3f}ms/{v[1]}" for k, v in p.items() if v[1]))
