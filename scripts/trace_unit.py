#!/usr/bin/env python3
"""Per-CTA timeline of the one-launch step kernel (decode_unit.cu, SKV_TRACE build): SM id and
globaltimer at each phase boundary, for the 8b-128k shapes (device residency), 2 layers."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["SKV_LIB"] = os.environ.get("SKV_TRACE_LIB") or os.path.join(ROOT, "paper_2504_00970_b200", "libsentencekv_trace.so")
import numpy as np, torch
import paper_2504_00970_b200 as skvlib, synth

SCRIPT = "script" in sys.argv[1:]  # the bench's decode script (boundary inputs, topic changes), 8 steps cycled
B, M, Hq, G, d, L, tau = 4, (8 if SCRIPT else 2), 32, 8, 128, 131072, 2048
dev = torch.device("cuda:0")
toks, topics = synth.prompts(0, B, L, 25.0)
HOST = "host" in sys.argv[1:]
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
buf = (ctypes.c_ulonglong * (1024 * 32))()
names = ["start", "scored", "csyncA", "bandpath", "general", "selected", "rowtab", "attended", "csync2", "end"]
if SCRIPT:
    script, target = synth.decode_script(0, B, 8)
    qpool = []
    for p in range(8):
        tg = torch.from_numpy(target[p]).to(dev)
        qpool.append([synth.queries_torch(gen, KV[l][2], tg, Hq, G, d).contiguous() for l in range(M)])
    itp = [torch.from_numpy(script[p]).to(dev) for p in range(8)]
    # one CUDA graph per pool step (all M layers), replayed as in bench.py
    for p in range(8):
        for l in range(M):
            skv.decode_step(l, qpool[p][l], itp[p], out)
    torch.cuda.synchronize()
    graphs = []
    st = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(st):
        for p in range(8):
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=st):
                for l in range(M):
                    skv.decode_step(l, qpool[p][l], itp[p], out)
            graphs.append(gr)
    torch.cuda.synchronize()
lbuf = (ctypes.c_ulonglong * (64 * 4))()
skvlib.lib.sentencekv_debug_launches(lbuf, 1)
for step in range(24 if SCRIPT else 10):
    if SCRIPT:
        if step == 23:
            skvlib.lib.sentencekv_debug_launches(lbuf, 1)
        graphs[step % 8].replay()
    for l in range(0 if SCRIPT else M):
        q = synth.queries_torch(gen, KV[l][2], tgt, Hq, G, d).contiguous()
        skv.decode_step(l, q, it, out)
    torch.cuda.synchronize()
    skvlib.lib.sentencekv_debug_unit(buf)
    T = np.array(buf, dtype=np.float64).reshape(1024, 32)[:n]
    sm = T[:, 23].astype(int)
    gen_path = T[:, 4] > T[:, 3]  # the general path stamps phase 4 after the band attempt
    T[~gen_path, 4] = T[~gen_path, 3]
    t = (T[:, :10] - T[:, 0].min()) / 1e3
    print(f"step {step}: span {t[:, 9].max():.2f} us; general-path CTAs {int(gen_path.sum())}/{n}; CTAs per SM: {np.bincount(np.bincount(sm, minlength=148))}")
    print("   phase        min    median   max  (us since first CTA start)")
    for i, nm in enumerate(names):
        print(f"   {nm:10s} {t[:, i].min():7.2f} {np.median(t[:, i]):7.2f} {t[:, i].max():7.2f}")
    reason = T[::8, 10].astype(int) & 15
    mode = (T[::8, 10].astype(int) >> 4) - 1
    print(f"   band modes per unit: { {m: int((mode == m).sum()) for m in (-1, 0, 2)} } (0 in band, 2 above the band, -1 general)")
    print(f"   band path per unit: reasons {np.bincount(reason, minlength=16)[:16].tolist()} (1 ovf, 2 above>tau, 4 below band, 8 nsel>cap); "
          f"band entries median {np.median(T[::8, 11]):.0f} max {T[::8, 11].max():.0f}; selected median {np.median(T[::8, 12]):.0f}; listed median {np.median(T[::8, 13]):.0f} max {T[::8,13].max():.0f}")
    sub = (T[:, [2, 16, 17, 18, 3]] - T[:, 0].min()) / 1e3
    ds = np.diff(sub, axis=1)
    print("   band sub-phases (median/max): " + ", ".join(f"{nm}={np.median(ds[:, i]):.2f}/{ds[:, i].max():.2f}" for i, nm in enumerate(["decide", "gather", "rank", "compact"])))
    if gen_path.any():
        gs = (T[gen_path][:, [4, 19, 20, 21, 5]] - T[:, 0].min()) / 1e3
        dg = np.diff(gs, axis=1)
        oc = T[gen_path][:, 14].astype(np.int64)
        print(f"   general: own candidates median {np.median(oc & 0xffffffff):.0f} max {(oc & 0xffffffff).max()}, in global {int((oc >> 32).sum())}; union median {np.median(T[gen_path][:, 15]):.0f} max {T[gen_path][:, 15].max():.0f}")
        print("   general sub-phases (median/max): " + ", ".join(f"{nm}={np.median(dg[:, i]):.2f}/{dg[:, i].max():.2f}" for i, nm in enumerate(["gather", "minmax", "levels", "compact"])))
    d_ = np.diff(t, axis=1)
    print("   durations (median/max): " + ", ".join(f"{names[i+1]}={np.median(d_[:, i]):.2f}/{d_[:, i].max():.2f}" for i in range(9)))

# per-launch: entry of the first CTA, first return from the programmatic-launch wait, last exit
torch.cuda.synchronize()
skvlib.lib.sentencekv_debug_launches(lbuf, 0)
Lt = np.array(lbuf, dtype=np.uint64).reshape(64, 4)
Lt = Lt[Lt[:, 0] != np.uint64(0xffffffffffffffff)].astype(np.float64)  # slots written since the reset
Lt = Lt[np.argsort(Lt[:, 0])]
n_l = len(Lt)
print("launches (us): entry->wait-return, wait-return->exit (span), previous exit->entry, previous exit->wait-return")
for i in range(1, n_l):
    print(f"  {i:3d} {(Lt[i,1]-Lt[i,0])/1e3:7.2f} {(Lt[i,2]-Lt[i,1])/1e3:7.2f} {(Lt[i,0]-Lt[i-1,2])/1e3:7.2f} {(Lt[i,1]-Lt[i-1,2])/1e3:7.2f}")
