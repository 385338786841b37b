#!/usr/bin/env python3
"""Per-CTA timeline of the one-launch step kernel (decode_unit.cu, SKV_TRACE build): SM id and
globaltimer at each phase boundary, for the 8b-128k shapes (device residency), 2 layers."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["SKV_LIB"] = os.environ.get("SKV_TRACE_LIB") or os.path.join(ROOT, "paper_2504_00970_b200", "libsentencekv_trace.so")
import numpy as np, torch
import paper_2504_00970_b200 as skvlib, synth

B, M, Hq, G, d, L, tau = 4, 2, 32, 8, 128, 131072, 2048
dev = torch.device("cuda:0")
toks, topics = synth.prompts(0, B, L, 25.0)
HOST = len(sys.argv) > 1 and sys.argv[1] == "host"
skv = skvlib.SentenceKV(batch=B, layers=M, q_heads=Hq, kv_heads=G, head_dim=d, max_context=L, token_budget=tau,
                        residency=skvlib.SKV_KV_HOST if HOST else skvlib.SKV_KV_DEVICE)
top = torch.from_numpy(topics).to(dev)
KV = [synth.kv_layer_torch(0, l, top, G, d, device=dev) for l in range(M)]
for l in range(M):
    skv.prefill_compress(l, KV[l][0], KV[l][1], torch.from_numpy(toks).to(dev) if l == 0 else None,
                         synth.BOUNDARY_IDS if l == 0 else None)
gen = torch.Generator(device=dev); gen.manual_seed(1)
tgt = torch.zeros(B, dtype=torch.int32, device=dev)
out = torch.empty((B, Hq, d), dtype=torch.float32, device=dev)
it = torch.full((B,), 300, dtype=torch.int32, device=dev)
n = B * G * 8
buf = (ctypes.c_ulonglong * (1024 * 24))()
names = ["start", "scored", "csyncA", "bandpath", "general", "selected", "rowtab", "attended", "csync2", "end"]
for step in range(10):
    for l in range(M):
        q = synth.queries_torch(gen, KV[l][2], tgt, Hq, G, d).contiguous()
        skv.decode_step(l, q, it, out)
    torch.cuda.synchronize()
    skvlib.lib.sentencekv_debug_unit(buf)
    T = np.array(buf, dtype=np.float64).reshape(1024, 24)[:n]
    sm = T[:, 23].astype(int)
    gen_path = T[:, 4] > T[:, 3]  # the general path stamps phase 4 after the band attempt
    T[~gen_path, 4] = T[~gen_path, 3]
    t = (T[:, :10] - T[:, 0].min()) / 1e3
    print(f"step {step}: span {t[:, 9].max():.2f} us; general-path CTAs {int(gen_path.sum())}/{n}; CTAs per SM: {np.bincount(np.bincount(sm, minlength=148))}")
    print("   phase        min    median   max  (us since first CTA start)")
    for i, nm in enumerate(names):
        print(f"   {nm:10s} {t[:, i].min():7.2f} {np.median(t[:, i]):7.2f} {t[:, i].max():7.2f}")
    reason = T[::8, 10].astype(int)
    print(f"   band path per unit: reasons {np.bincount(reason, minlength=16)[:16].tolist()} (1 ovf, 2 above>tau, 4 below band, 8 nsel>cap); "
          f"band entries median {np.median(T[::8, 11]):.0f} max {T[::8, 11].max():.0f}; selected median {np.median(T[::8, 12]):.0f}; listed median {np.median(T[::8, 13]):.0f} max {T[::8,13].max():.0f}")
    sub = (T[:, [2, 16, 17, 18, 3]] - T[:, 0].min()) / 1e3
    ds = np.diff(sub, axis=1)
    print("   band sub-phases (median/max): " + ", ".join(f"{nm}={np.median(ds[:, i]):.2f}/{ds[:, i].max():.2f}" for i, nm in enumerate(["decide", "gather", "rank", "compact"])))
    if gen_path.any():
        gs = (T[gen_path][:, [4, 19, 20, 21, 5]] - T[:, 0].min()) / 1e3
        dg = np.diff(gs, axis=1)
        print("   general sub-phases (median/max): " + ", ".join(f"{nm}={np.median(dg[:, i]):.2f}/{dg[:, i].max():.2f}" for i, nm in enumerate(["gather", "minmax", "levels", "compact"])))
    d_ = np.diff(t, axis=1)
    print("   durations (median/max): " + ", ".join(f"{names[i+1]}={np.median(d_[:, i]):.2f}/{d_[:, i].max():.2f}" for i in range(9)))
