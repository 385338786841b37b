#!/usr/bin/env python3
"""How much of a decode step's selection is predictable from the previous step's, under the bench's
conditions (8b-128k shapes, device residency, fresh decode-script queries, topic switch after each
boundary input).  For each (layer, unit) and step: with the previous step's lowest selected key ks
and crossing key kc (ordered 32-bit keys of the scores), and a margin w, the sentences with key >
k_spec (= ks + w or kc + w) are certainly selected iff their total length <= tau.  Prints, per rule
and margin, the share of the selected tokens above k_spec (0 when the rule fails) and how often it
fails.  Usage: spec_probe.py [layers] [steps]"""
import os, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2504_00970_b200 as skvlib, synth

M = int(sys.argv[1]) if len(sys.argv) > 1 else 2
STEPS = int(sys.argv[2]) if len(sys.argv) > 2 else 60
B, Hq, G, d, L, tau = 4, 32, 8, 128, 131072, 2048
dev = torch.device("cuda:0")
toks, topics = synth.prompts(0, B, L, 25.0)
skv = skvlib.SentenceKV(batch=B, layers=M, q_heads=Hq, kv_heads=G, head_dim=d, max_context=L, token_budget=tau)
top = torch.from_numpy(topics).to(dev)
KV = []
for l in range(M):
    K, V, c = synth.kv_layer_torch(0, l, top, G, d, device=dev)
    skv.prefill_compress(l, K, V, torch.from_numpy(toks).to(dev) if l == 0 else None,
                         synth.BOUNDARY_IDS if l == 0 else None)
    skv.sync()
    KV.append((K, V, c))
S = torch.tensor(skv.sentence_counts(), device=dev)
off = skv.offsets()
Smax = off.shape[1] - 1
lens = (off[:, 1:] - off[:, :-1]).clamp(min=0).to(torch.int64)  # [B][Smax]
valid_s = torch.arange(Smax, device=dev)[None, :] < S[:, None]


def okey(x):  # ordered 32-bit key of an fp32 score (as int64)
    u = x.contiguous().view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    u = torch.where((u & 0x7FFFFFFF) == 0, torch.zeros_like(u), u)
    neg = (u >> 31) == 1
    return torch.where(neg, (~u) & 0xFFFFFFFF, u | 0x80000000)


script, target = synth.decode_script(0, B, STEPS + 1)
gen = torch.Generator(device=dev)
gen.manual_seed(1)
out = torch.empty((B, Hq, d), dtype=torch.float32, device=dev)
ids = torch.empty((B, G, tau), dtype=torch.int32, device=dev)
margins = [0, 1 << 14, 1 << 16, 1 << 17, 1 << 18, 1 << 19]
acc = {(r, m): [0.0, 0, 0] for r in ("ks", "kc") for m in margins}  # share sum, fails, samples
prev = [None] * M
for step in range(STEPS):
    tg = torch.from_numpy(target[step]).to(dev)
    it = torch.from_numpy(script[step]).to(dev)
    for l in range(M):
        q = synth.queries_torch(gen, KV[l][2], tg, Hq, G, d).contiguous()
        skv.decode_step(l, q, it, out, ids)
        sc = skv.scores(l)  # [B][G][Smax]
        k = okey(sc)
        sel = torch.zeros((B, G, Smax + 1), dtype=torch.bool, device=dev)
        idx = ids.to(torch.int64).clamp(min=-1) + 1  # -1 padding -> column 0, dropped below
        sel.scatter_(2, idx, True)
        sel = sel[:, :, 1:] & valid_s[:, None, :]
        big = torch.iinfo(torch.int64).max
        ks = torch.where(sel, k, torch.full_like(k, big)).amin(dim=2)  # lowest selected key
        kc = torch.where(~sel & valid_s[:, None, :], k, torch.full_like(k, -1)).amax(dim=2)  # crossing
        ntok = (lens[:, None, :] * sel).sum(dim=2).clamp(min=1)
        if prev[l] is not None and step >= 5:
            pks, pkc = prev[l]
            for r, base in (("ks", pks), ("kc", pkc)):
                for m in margins:
                    above = (k > (base + m)[:, :, None]) & valid_s[:, None, :]
                    w = (lens[:, None, :] * above).sum(dim=2)
                    ok = w <= tau
                    share = torch.where(ok, w.double() / ntok.double(), torch.zeros_like(w, dtype=torch.float64))
                    a = acc[(r, m)]
                    a[0] += float(share.sum())
                    a[1] += int((~ok).sum())
                    a[2] += share.numel()
        prev[l] = (ks, kc)
print(f"layers {M}, steps {STEPS} (first 5 skipped), units {B * G}")
print("rule  margin   share of selected tokens above k_spec   fail rate")
for (r, m), (s, f, n) in acc.items():
    print(f"{r:4s}  2^{int(np.log2(m)) if m else '-':<4}  {s / n:8.3f}                              {f / n:7.3f}")
