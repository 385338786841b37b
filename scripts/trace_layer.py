#!/usr/bin/env python3
"""Timeline of the persistent per-layer kernel's work items (SKV_TRACE build): claim / end times
per item kind, relative to the first claim of the launch."""
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
S = skv.sentence_counts()
n_score = [max(1, (s + 511) // 512) for s in S]
kinds = []
group = 8
units = B * G
ng = (units + group - 1) // group
for u in range(units):
    kinds += [("S", u)] * n_score[u // G]
kinds += [("L", u) for u in range(units)]
for i in range(tau // 256):
    kinds += [("A", u) for u in range(units)]
n = len(kinds)
buf = (ctypes.c_ulonglong * (2 * n))()
for step in range(4):
    for l in range(M):
        q = synth.queries_torch(gen, KV[l][2], tgt, Hq, G, d).contiguous()
        skv.decode_step(l, q, it, out)
    torch.cuda.synchronize()
skvlib.lib.sentencekv_debug_items(buf, n)
t = np.array(buf, dtype=np.float64).reshape(n, 2)
t0 = t[:, 0].min()
t = (t - t0) / 1e3
print(f"items {n}, launch span {t[:, 1].max():.2f} us")
for kind in "SLA":
    idx = [i for i, (kk, _) in enumerate(kinds) if kk == kind]
    st, en = t[idx, 0], t[idx, 1]
    print(f"{kind}: n={len(idx)} first claim {st.min():.2f} last claim {st.max():.2f} first end {en.min():.2f} "
          f"last end {en.max():.2f} mean dur {np.mean(en - st):.2f} max dur {np.max(en - st):.2f}")
for gi in range(ng):
    for kind in "SLA":
        idx = [i for i, (kk, u) in enumerate(kinds) if kk == kind and u // group == gi]
        print(f"  group {gi} {kind}: claim [{t[idx,0].min():.1f}, {t[idx,0].max():.1f}] end [{t[idx,1].min():.1f}, {t[idx,1].max():.1f}]")

ph = (ctypes.c_ulonglong * (64 * 16))()
skvlib.lib.sentencekv_debug_phases(ph)
P = np.array(ph, dtype=np.float64).reshape(64, 16)
print("SELECT phases (us from item start): wait, loadcands, -, range, select, compact, release")
for u in range(0, units, 4):
    r = P[u, :8]
    print(u, " ".join(f"{(r[i]-r[0])/1e3:.2f}" for i in range(1, 8)), f"| item start {(r[0]-t0)/1e3:.2f}")
