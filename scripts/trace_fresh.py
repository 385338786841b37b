#!/usr/bin/env python3
"""Per-launch phase timeline of the step kernel (SKV_TRACE build) under the bench's conditions:
8b-128k shapes, FRESH queries every step from the seeded decode script (topic switch after each
boundary input), eager decode_step per layer.  Usage: trace_fresh.py [host|device] [layers] [steps]"""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["SKV_LIB"] = os.environ.get("SKV_TRACE_LIB") or os.path.join(ROOT, "paper_2504_00970_b200", "libsentencekv_trace.so")
import numpy as np, torch
import paper_2504_00970_b200 as skvlib, synth

HOST = (sys.argv[1] if len(sys.argv) > 1 else "host") == "host"
RET = (sys.argv[1] if len(sys.argv) > 1 else "") == "ret"  # device residency + NEXT-1 retention (N = 32)
M = int(sys.argv[2]) if len(sys.argv) > 2 else 4
STEPS = int(sys.argv[3]) if len(sys.argv) > 3 else 60
B, Hq, G, d, L, tau = 4, 32, 8, 128, 131072, 2048
dev = torch.device("cuda:0")
toks, topics = synth.prompts(0, B, L, 25.0)
skv = skvlib.SentenceKV(batch=B, layers=M, q_heads=Hq, kv_heads=G, head_dim=d, max_context=L, token_budget=tau,
                        residency=skvlib.SKV_KV_HOST if HOST else skvlib.SKV_KV_DEVICE, obs_window=32 if RET else 0)
wg = torch.Generator(device=dev)
top = torch.from_numpy(topics).to(dev)
KV = []
for l in range(M):
    K, V, c = synth.kv_layer_torch(0, l, top, G, d, device=dev)
    qw = None
    if RET:
        wg.manual_seed(4242 + 7919 * l)
        qw = synth.window_queries_torch(wg, c, top[:, L - 32:], Hq, G, d).contiguous()
    skv.prefill_compress(l, K, V, torch.from_numpy(toks).to(dev) if l == 0 else None, synth.BOUNDARY_IDS if l == 0 else None, q_window=qw)
    skv.sync()
    KV.append((None, None, c) if (HOST or RET) else (K, V, c))
script, target = synth.decode_script(0, B, STEPS + 1)
gen = torch.Generator(device=dev); gen.manual_seed(1)
out = torch.empty((B, Hq, d), dtype=torch.float32, device=dev)
n = B * G * 8
buf = (ctypes.c_ulonglong * (1024 * 32))()
rows = []
why = []
for step in range(STEPS):
    tg = torch.from_numpy(target[step]).to(dev)
    it = torch.from_numpy(script[step]).to(dev)
    led0 = [skv.host_fetch_bytes(l) for l in range(M)]
    for l in range(M):
        q = synth.queries_torch(gen, KV[l][2], tg, Hq, G, d).contiguous()
        torch.cuda.synchronize()
        skv.decode_step(l, q, it, out)
        torch.cuda.synchronize()
        skvlib.lib.sentencekv_debug_unit(buf)
        T = np.array(buf, dtype=np.float64).reshape(1024, 32)[:n]
        t0 = T[:, 0].min()
        t = lambda i: (T[:, i] - t0) / 1e3
        miss = T[:, 24] > 0
        gen_path = T[:, 4] > T[:, 3]
        hb = (skv.host_fetch_bytes(l) - led0[l]) if HOST else 0
        reason = T[::8, 10].astype(int) & 15
        for u in np.nonzero(gen_path[::8])[0]:
            why.append((step, l, int(u), int(reason[u]), int(T[u * 8, 13])))
        bandp = ~gen_path
        sub = {}
        if bandp.any():
            for nm, (x0, x1) in (("b_decide", (2, 16)), ("b_gather", (16, 17)), ("b_rank", (17, 18)), ("b_compact", (18, 3))):
                sub[nm] = float(np.max(t(x1)[bandp] - t(x0)[bandp]))
        if gen_path.any():
            for nm, (x0, x1) in (("g_local", (3, 4)), ("g_gather", (4, 19)), ("g_minmax", (19, 20)), ("g_levels", (20, 21)), ("g_compact", (21, 5))):
                sub[nm] = float(np.max(t(x1)[gen_path] - t(x0)[gen_path]))
        rows.append(dict(step=step, layer=l, span=t(9).max(), **sub, scored=t(1).max(), selected=t(5).max(),
                         rowtab=t(25).max(), planned=t(6).max(), attended=t(7).max(), csync2=t(8).max(),
                         miss_ctas=int(miss.sum()), gen_ctas=int(gen_path.sum()), host_mb=hb / 1e6,
                         att_miss=np.median(t(7)[miss] - t(6)[miss]) if miss.any() else 0.0,
                         plan_miss=np.median(t(6)[miss] - t(25)[miss]) if miss.any() else 0.0,
                         att_hit=np.median(t(7)[~miss] - t(6)[~miss]) if (~miss).any() else 0.0,
                         **({f"p{k}": float(np.median(t(k)[miss] - t(k - 1 if k > 26 else 25)[miss])) for k in (26, 27, 28, 29, 30)}
                            if miss.any() else {f"p{k}": 0.0 for k in (26, 27, 28, 29, 30)})))
import statistics as st
keys = ["span", "scored", "selected", "rowtab", "planned", "attended", "csync2", "miss_ctas", "gen_ctas", "host_mb", "plan_miss", "att_miss", "att_hit", "p26", "p27", "p28", "p29", "p30",
        "b_decide", "b_gather", "b_rank", "b_compact", "g_local", "g_gather", "g_minmax", "g_levels", "g_compact"]
print(f"residency={'host' if HOST else 'device'}{' +retention' if RET else ''} layers={M} steps={STEPS}: per launch (max over CTAs of phase end, us since first CTA start)")
med = lambda rs, k: st.median([r[k] for r in rs if k in r]) if any(k in r for r in rs) else float("nan")
print("  all  : " + " ".join(f"{k}={med(rows, k):.2f}" for k in keys))
for sel, name in ((lambda r: r["miss_ctas"] == 0, "nomiss"), (lambda r: 0 < r["miss_ctas"] and r["host_mb"] < 1, "fewmiss"), (lambda r: r["host_mb"] >= 1, "bigmiss")):
    rs = [r for r in rows if sel(r)]
    if rs:
        print(f"  {name:6s} n={len(rs):4d}: " + " ".join(f"{k}={med(rs, k):.2f}" for k in keys))
from collections import Counter
late = [w for w in why if w[0] > 0]
print("general-path units after step 0:", len(late), "of", (STEPS - 1) * M * B * G, "unit-launches; reasons (1 ovf, 2 above>tau, 4 below band):",
      dict(Counter(w[3] for w in late)), "; units per launch:", dict(Counter(Counter((w[0], w[1]) for w in late).values())))
print("  first 30:", late[:30])
print("per step span sum (us):", [round(sum(r["span"] for r in rows if r["step"] == s), 1) for s in range(STEPS)])
