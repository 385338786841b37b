#!/usr/bin/env python
"""bench.py -- SentenceKV decode-step benchmark on B200 (driver contract: one JSON line on rank 0).

A "step" is one pass of the whole hot path for one decode token of every sequence: for every layer
one sentencekv_decode_step (D1 Eq. 2 query cache + scores over all sentence embeddings, D2 budgeted
whole-sentence selection, D3 gather, D4 Eq. 3 attention), captured once into a CUDA graph.  Prefill
(P1 segmentation, P2 embeddings, P3 offload in host residency) runs once before the timed region.

Every timed step gets FRESH inputs: the queries and input tokens of step k of a seeded decode
script (a boundary input about every 25 steps per sequence, after which the query topic changes,
synth.decode_script) are copied into the graph's static input buffers before its replay (the 1 MB
device-to-device copy is inside the timed region).  In host residency the topic switches make the
selection move, so the per-step host-link traffic of D3 is the real one ("onload
1024 tokens 0.0038 s" is the paper's cost of that transfer on H100 + PCIe).

Default workload (BASELINE.json metric "decode-step latency (ms) & tokens/s at 128K ctx"):
configs[2] = Llama-3.1-8B shapes (32 layers, 32 Q / 8 KV heads, d=128), 128K context, tau=2048,
batch 4, full K/V offloaded to pinned host.  value = tokens/s = sequences decoded per second (B per
step) over all ranks.  --config 8b-32k / 8b-256k give the configs[1] / configs[3] lines.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 8b-128k] [--impl ours|reference]

Multi-GPU (torchrun, one process per GPU): --shard heads (default) splits the KV heads (then the
batch) of the fixed global batch over the ranks -- strong scaling -- with one NCCL all-gather of the
per-head outputs per layer inside the captured step; --shard batch gives every rank its own batch
(weak scaling, device residency only: the host store would not fit the box's RAM at 8 ranks).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (B, M layers, Hq, G, d, L, tau, median sentence length)
    "tiny": dict(B=1, M=1, Hq=8, G=2, d=64, L=4096, tau=256, median=20.0),
    "8b-32k": dict(B=1, M=32, Hq=32, G=8, d=128, L=32768, tau=1024, median=25.0),
    "8b-128k": dict(B=4, M=32, Hq=32, G=8, d=128, L=131072, tau=2048, median=25.0),
    "8b-256k": dict(B=1, M=32, Hq=32, G=8, d=128, L=262144, tau=4096, median=25.0),
    "70b-128k": dict(B=16, M=80, Hq=64, G=8, d=128, L=131072, tau=2048, median=25.0),
}
METRIC = "decode-step latency (ms) & tokens/s at 128K ctx; achieved HBM GB/s vs B200 peak"
SEED = 0
CHECK_UNITS = 4  # (layer, b, g) units checked against the oracle at the end of the timed run


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="8b-128k", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-split", action="store_true", help="skip the decode_select + decode_attend line")
    ap.add_argument("--no-check", action="store_true", help="skip the end-of-run oracle check")
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--shard", choices=["heads", "batch"], default="heads")
    ap.add_argument("--gather", choices=["nccl", "fused"], default="nccl",
                    help="N > 1: the per-layer output all-gather by NCCL (default) or fused into the attention "
                         "epilogue (peer stores into torch symmetric memory + arrival counters, SURVEY 8(e))")
    ap.add_argument("--retention", action="store_true",
                    help="NEXT-1: importance-filtered retention at prefill (observation window of --obs-window "
                         "queries, top floor(r*tau) tokens kept in an HBM pool); decode ranks and attends the pool")
    ap.add_argument("--obs-window", type=int, default=32)
    ap.add_argument("--buckets", choices=["sentence", "equal", "quest"], default="sentence",
                    help="NEXT-3 equal-size chunks / NEXT-4 Quest pages instead of sentences")
    ap.add_argument("--page", type=int, default=16, help="Quest page size (tokens)")
    ap.add_argument("--outlier-n", type=float, default=0.0, help="NEXT-3 outlier split at mean + n*std (0 = off)")
    ap.add_argument("--query", choices=["mean", "current"], default="mean", help="NEXT-3 current-token query")
    ap.add_argument("--fill", choices=["prefix", "skip"], default="prefix", help="NEXT-3 skip-and-continue fill")
    ap.add_argument("--local", action="store_true",
                    help="NEXT-2: every step appends the token's K/V (local segment, context growth)")
    ap.add_argument("--residency", choices=["device", "host"], default=None,
                    help="K/V residency (default: host for 8b-128k, which configs[2] specifies, else device)")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def config_dict(args, cfg, GB, extra=None):
    tags = [t for t, on in (("retention", getattr(args, "retention", False)),
                            (f"{getattr(args, 'buckets', 'sentence')}" + (f"{args.page}" if getattr(args, "buckets", "") == "quest" else ""),
                             getattr(args, "buckets", "sentence") != "sentence"),
                            (f"outlier{getattr(args, 'outlier_n', 0)}", getattr(args, "outlier_n", 0) > 0),
                            ("current-query", getattr(args, "query", "mean") == "current"),
                            ("skip-fill", getattr(args, "fill", "prefix") == "skip"),
                            ("local", getattr(args, "local", False))) if on]
    d = {"workload": "+".join([args.config] + tags), "global_batch": GB, "layers": cfg["M"], "q_heads": cfg["Hq"],
         "kv_heads": cfg["G"], "head_dim": cfg["d"], "context": cfg["L"], "token_budget": cfg["tau"],
         "median_sentence_tokens": cfg["median"]}
    d.update(extra or {})
    return d


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML in a thread during the timed region."""

    def __init__(self, index: int, period_s: float = 0.01):
        self.index, self.period = index, period_s
        self.sm, self.reasons, self.max_sm = [], set(), None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.nv = pynvml
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception as e:  # NVML missing: record it
            self.reasons.add(f"nvml_unavailable:{type(e).__name__}")
        return self

    def _run(self):
        nv = self.nv
        names = {0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
                 0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
                 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}
        while not self._stop.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in names.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.max_sm,
                "reasons": sorted(self.reasons), "samples": len(self.sm)}


def pct(xs, p):
    return float(np.percentile(np.asarray(xs), p)) if len(xs) else None


# --------------------------------------------------------------------------- oracle timing


class OracleStep:
    """The CPU oracle (tests' checker, oracle/) driven over full decode steps of a workload: every
    layer, every (b, g) unit, select (Eq. 2 + scores + budgeted selection) + attend (Eq. 3), units
    in parallel on all host threads (the C functions release the GIL).  K/V host copies exist for
    `kv_layers` layers; layer l of a step uses the bytes of layer l % len(kv_layers) (same shapes,
    same work), its own queries."""

    def __init__(self, cfg, toks, Kh, Vh):
        import oracle
        import synth

        self.oracle, self.synth = oracle, synth
        self.cfg = cfg
        self.G, self.Hq, self.d, self.tau, self.M = cfg["G"], cfg["Hq"], cfg["d"], cfg["tau"], cfg["M"]
        self.grp = self.Hq // self.G
        self.B = toks.shape[0]
        self.Kh, self.Vh = Kh, Vh  # lists of uint16 [B][G][L][d]
        self.threads = len(os.sched_getaffinity(0))
        import concurrent.futures as cf

        self.ex = cf.ThreadPoolExecutor(self.threads)
        self.off = [oracle.segment(toks[b], synth.BOUNDARY_IDS, self.tau) for b in range(self.B)]
        futs = {(i, b, g): self.ex.submit(oracle.embed, Kh[i][b, g], self.off[b])
                for i in range(len(Kh)) for b in range(self.B) for g in range(self.G)}
        self.E = {k: f.result() for k, f in futs.items()}
        self.Sq = np.zeros((self.M, self.B, self.Hq, self.d), np.float32)
        self.cnt = np.zeros((self.M, self.B), np.int32)
        self.bset = set(synth.BOUNDARY_IDS.tolist())

    def step(self, q_layers, itok):
        """One full decode step.  q_layers[l]: uint16 [B][Hq][d]; itok int32 [B]."""
        o = self.oracle
        nkv = len(self.Kh)

        def unit(l, b, g, qbar):
            i = l % nkv
            qt = o.group_query(qbar, self.grp, g)
            sc = o.score(qt, self.E[(i, b, g)])
            ids, _ = o.select(sc, self.off[b], self.tau)
            return o.attend(q_layers[l][b, g * self.grp:(g + 1) * self.grp], self.Kh[i][b, g], self.Vh[i][b, g],
                            self.off[b], ids)

        futs = []
        for l in range(self.M):
            for b in range(self.B):
                qbar = o.qs_append_mean(self.Sq[l, b], self.cnt[l, b:b + 1], q_layers[l][b])
                futs += [self.ex.submit(unit, l, b, g, qbar) for g in range(self.G)]
                if int(itok[b]) in self.bset:
                    o.qs_reset(self.Sq[l, b], self.cnt[l, b:b + 1])
        for f in futs:
            f.result()


def time_oracle(ost, qsteps, itoks, n_steps, budget_s=None):
    """Times n_steps full oracle steps (or as many as fit budget_s after the first).  Returns
    (seconds per step list)."""
    times = []
    for k in range(n_steps):
        t0 = time.perf_counter()
        ost.step(qsteps[k % len(qsteps)], itoks[k % len(itoks)])
        times.append(time.perf_counter() - t0)
        if budget_s is not None and sum(times) >= budget_s:
            break
    return times


# --------------------------------------------------------------------------- main


def main():
    args = parse()
    residency = args.residency or ("host" if args.config in ("8b-128k",) and not args.retention else "device")
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: SKV_BENCH_SAME_GPU=1 puts every rank on cuda:0 with the gloo backend, so the N > 1
    # code path (shards, per-layer all-gather, barriers, max over ranks) can be exercised on one GPU;
    # never used for a reported number
    same_gpu = os.environ.get("SKV_BENCH_SAME_GPU", "") == "1"
    if same_gpu:
        local = 0
    cfg = dict(CONFIGS[args.config])
    B, M, Hq, G, d, L, tau = (cfg[k] for k in ("B", "M", "Hq", "G", "d", "L", "tau"))
    hbm_peak, peak_kind = peaks()
    if args.impl == "reference":
        return reference_arm(args, cfg, rank, world, residency)

    import torch
    import torch.distributed as dist

    import synth

    if args.retention and world > 1 and args.shard != "batch":
        raise SystemExit("--retention sums alpha over all heads (P:394): shard by batch (--shard batch)")
    if args.shard == "batch" and residency == "host" and world > 1:
        raise SystemExit("--shard batch with host residency would pin world x the host store; use --shard heads")
    if world > 1:
        torch.cuda.set_device(local)
        if same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    import paper_2504_00970_b200 as skvlib
    from paper_2504_00970_b200 import parallel

    GB = B * world if args.shard == "batch" else B  # global batch
    plan = parallel.plan(GB, G, Hq, world, rank, "batch" if args.shard == "batch" else "heads")
    Bl, Gl, Hl = plan.batch_count, plan.kv_head_count, plan.q_head_count
    b0, g0, h0 = plan.batch_begin, plan.kv_head_begin, plan.q_head_begin
    plain = (not args.retention and args.buckets == "sentence" and args.outlier_n == 0 and args.query == "mean"
             and args.fill == "prefix" and not args.local)
    cpu_leg = rank == 0 and world == 1 and not args.no_cpu_baseline and plain
    check = rank == 0 and world == 1 and not args.no_check and plain
    N = args.obs_window if args.retention else 0
    keep_layers = [0, 1][:M] if (cpu_leg or check) else []

    # ---------------- inputs (seeded, synthetic; this rank's shard of sequences and heads)
    toks, topics = zip(*(synth.token_stream(SEED, b0 + b, L, cfg["median"]) for b in range(Bl)))
    toks, topics = np.stack(toks), np.stack(topics)
    tok_dev = torch.from_numpy(toks).to(dev)
    top_dev = torch.from_numpy(topics).to(dev)
    host = residency == "host"
    n_cold_, n_split_ = (1 if residency == "host" else 0), (0 if args.no_split else 1 + max(2, args.warmup) + min(args.steps, 100))
    max_gen = (n_cold_ + 2 + max(1, args.warmup) + args.steps + 1 + 4 + n_split_ + args.e2e_steps + 8) if args.local else 0
    variant = dict(max_generated=max_gen, bucket_mode={"sentence": 0, "equal": 1, "quest": 2}[args.buckets],
                   chunk_size=args.page if args.buckets == "quest" else 0, outlier_n=args.outlier_n,
                   query_mode=1 if args.query == "current" else 0, fill_mode=1 if args.fill == "skip" else 0)
    skv = skvlib.SentenceKV(layers=M, head_dim=d, max_context=L, token_budget=tau, device=local,
                            residency=skvlib.SKV_KV_HOST if host else skvlib.SKV_KV_DEVICE, obs_window=N,
                            **variant, **plan.ctx_kwargs())
    wgen = torch.Generator(device=dev)
    # ---------------- K/V generation + prefill (P1 segmentation, P2 embeddings, P3 offload in host
    # residency), per layer; in host residency the device K/V of a layer is freed once offloaded
    # (layers 0, 1 are copied to the host for the CPU oracle's baseline and end-of-run check).
    # load the prefill kernels once (CUDA loads a module's kernels lazily at their first launch; that
    # one-time host cost must not land in the prefill timings below)
    warm = skvlib.SentenceKV(batch=1, layers=1, q_heads=Hq, kv_heads=G, head_dim=d, max_context=128, token_budget=64,
                             device=local, obs_window=(16 if N else 0), **{k: v for k, v in variant.items() if k != "max_generated"})
    wk = torch.zeros((1, G, 128, d), dtype=torch.bfloat16, device=dev)
    warm.prefill_compress(0, wk, wk, token_ids=torch.zeros((1, 128), dtype=torch.int32, device=dev),
                          boundary_ids=synth.BOUNDARY_IDS,
                          q_window=torch.zeros((1, 16, Hq, d), dtype=torch.bfloat16, device=dev) if N else None)
    warm.sync()
    warm.close()
    Ks, Vs, Cs, Kh, Vh = [], [], [], [], []
    t_gen = prefill_ms = offload_s = 0.0
    skv.set_profiling(True)
    for l in range(M):
        t0 = time.perf_counter()
        K, V, c = synth.kv_layer_torch(SEED, l, top_dev, G, d, device=dev, b_begin=b0, g_begin=g0, g_count=Gl)
        torch.cuda.synchronize()
        t_gen += time.perf_counter() - t0
        pf0 = torch.cuda.Event(enable_timing=True)
        pf1 = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        pf0.record()
        qw = None
        if N:  # the window's own queries: about the topics of the last N prompt tokens
            wgen.manual_seed(4242 + 7919 * l)
            qw = synth.window_queries_torch(wgen, c, top_dev[:, L - N:], Hq, G, d)[:, :, h0:h0 + Hl].contiguous()
        skv.prefill_compress(l, K, V, token_ids=tok_dev if l == 0 else None,
                             boundary_ids=synth.BOUNDARY_IDS if l == 0 else None, q_window=qw)
        pf1.record()
        if host:
            skv.sync()  # D2H copies of this layer done
            offload_s += time.perf_counter() - t0
        torch.cuda.synchronize()
        prefill_ms += pf0.elapsed_time(pf1)
        if l in keep_layers:
            Kh.append(K.view(torch.int16).cpu().numpy().view(np.uint16))
            Vh.append(V.view(torch.int16).cpu().numpy().view(np.uint16))
        Ks.append(None if (host or N) else K)  # host store / retained pool: the ctx keeps its own copy
        Vs.append(None if (host or N) else V)
        Cs.append(c)
        del K, V
    prof_prefill = skv.profile_read()
    skv.set_profiling(False)
    S = skv.sentence_counts()
    kv_bytes_total = 2 * Bl * Gl * L * d * 2 * M
    ret = None
    if N:  # buckets per layer (sentences with a retained token) replace the prompt's sentences
        Sl = [skv.retained(l)[3].cpu().numpy() for l in range(M)]
        ret = {"obs_window": N, "retained_tokens_per_seq": skv.retained_tokens(0),
               "buckets_mean_per_seq": round(float(np.mean([x.mean() for x in Sl])), 1),
               "retain_ms_per_layer": round(prof_prefill["retain"][0] / max(1, prof_prefill["retain"][1]), 4),
               "compress_ms_per_layer": round(prof_prefill["compress"][0] / max(1, prof_prefill["compress"][1]), 4)}
        S = [int(round(float(np.mean([x[b] for x in Sl])))) for b in range(Bl)]

    # ---------------- decode script: one fresh step of queries + input tokens per executed step
    n_cold, n_eager = (1 if host else 0), 2
    n_split = 0 if args.no_split else 1 + max(2, args.warmup) + min(args.steps, 100)  # eager + warm-up + timed
    n_prof = 4
    NQ = n_cold + n_eager + max(1, args.warmup) + args.steps + 1 + n_prof + n_split
    script, target = synth.decode_script(SEED, GB, NQ)
    script, target = script[:, b0:b0 + Bl].copy(), target[:, b0:b0 + Bl].copy()
    tgt = torch.from_numpy(target).to(dev)
    gen = torch.Generator(device=dev)
    qall = torch.empty((NQ, M, Bl, Hl, d), dtype=torch.bfloat16, device=dev)
    for l in range(M):
        cl = Cs[l][:, tgt.long(), :]                            # [G][NQ][Bl][d]
        cl = cl.permute(1, 2, 0, 3).repeat_interleave(Hq // G, dim=2)[:, :, h0:h0 + Hl]  # [NQ][Bl][Hl][d]
        gen.manual_seed(1234 + 104729 * l + 7919 * rank)
        qall[:, l] = (cl + torch.randn(cl.shape, generator=gen, device=dev)).to(torch.bfloat16)
    tall = torch.from_numpy(script).to(dev)                     # [NQ][Bl]
    kvall = None
    if args.local:  # NEXT-2: this step's generated K/V per layer, drawn like the context's (topic + noise)
        kvall = torch.empty((NQ, M, 2, Bl, Gl, d), dtype=torch.bfloat16, device=dev)
        for l in range(M):
            gen.manual_seed(777 + 104729 * l + 7919 * rank)
            cl = Cs[l][g0:g0 + Gl][:, tgt.long(), :].permute(1, 2, 0, 3)  # [NQ][Bl][Gl][d]
            kvall[:, l, 0] = (cl + torch.randn(cl.shape, generator=gen, device=dev)).to(torch.bfloat16)
            kvall[:, l, 1] = torch.randn(cl.shape, generator=gen, device=dev).to(torch.bfloat16)
    kvbuf = torch.empty((M, 2, Bl, Gl, d), dtype=torch.bfloat16, device=dev) if args.local else None
    qbuf = torch.empty((M, Bl, Hl, d), dtype=torch.bfloat16, device=dev)  # static inputs of the graph
    tbuf = torch.empty((Bl,), dtype=torch.int32, device=dev)
    outs = torch.empty((M, Bl, Hl, d), dtype=torch.float32, device=dev)
    gath = [torch.empty((world, Bl, Hl, d), dtype=torch.float32, device=dev) for _ in range(M)] if world > 1 else None
    fused = world > 1 and args.gather == "fused"
    if fused:
        # every rank's gather buffers and arrival counters in symmetric memory; the kernels store their
        # outputs into every peer's buffer and count arrivals (sentencekv_set_output_peers)
        import torch.distributed._symmetric_memory as symm_mem

        gbuf = symm_mem.empty((M, world, Bl, Hl, d), dtype=torch.float32, device=dev)
        fbuf = symm_mem.empty((M,), dtype=torch.int32, device=dev)
        fbuf.zero_()
        hb = symm_mem.rendezvous(gbuf, dist.group.WORLD)
        hf = symm_mem.rendezvous(fbuf, dist.group.WORLD)
        dist.barrier()
        lay = world * Bl * Hl * d * 4
        for l in range(M):
            skv.set_output_peers(l, rank, [hb.buffer_ptrs[p] + l * lay for p in range(world)],
                                 [hf.buffer_ptrs[p] + 4 * l for p in range(world)])
        gath = [gbuf[l] for l in range(M)]
    sel_tok = torch.zeros((M, Bl, Gl), dtype=torch.int32, device=dev)
    history = []  # script index of every decode step executed on the context, in order
    nxt = [0]

    def take():
        k = nxt[0]
        nxt[0] += 1
        history.append(k)
        return k

    def load(k):
        qbuf.copy_(qall[k], non_blocking=True)
        tbuf.copy_(tall[k], non_blocking=True)
        if kvbuf is not None:
            kvbuf.copy_(kvall[k], non_blocking=True)

    def body(with_tokens=False, split=False):
        for l in range(M):
            if kvbuf is not None:  # NEXT-2: the token's K/V joins the local segment before its attention
                skv.decode_append(l, kvbuf[l, 0], kvbuf[l, 1], tbuf)
            if split:
                skv.decode_select(l, qbuf[l], tbuf, sel_tokens=sel_tok[l] if with_tokens else None)
                skv.decode_attend(l, qbuf[l], outs[l])
            else:
                skv.decode_step(l, qbuf[l], tbuf, outs[l], sel_tokens=sel_tok[l] if with_tokens else None)
            if fused:  # the exchange happened in the kernel's epilogue: wait for every rank's arrivals
                skv.wait_outputs(l)
            elif world > 1:  # the one exchange: all-gather of the per-head outputs of the layer
                parallel.all_gather_outputs(outs[l], plan, gathered=gath[l])

    # cold step (host residency): the first decode step after the prefill finds the HBM page cache
    # empty, so every selected row of every layer crosses the host link (D3 host) -- its
    # device time and ledger bytes give the offload fetch's host-link GB/s
    cold = None
    if host:
        led0 = sum(skv.host_fetch_bytes(l) for l in range(M))
        load(take())
        torch.cuda.synchronize()
        c0 = torch.cuda.Event(enable_timing=True)
        c1 = torch.cuda.Event(enable_timing=True)
        c0.record()
        body()
        c1.record()
        torch.cuda.synchronize()
        cold_ms = c0.elapsed_time(c1)
        cold_bytes = sum(skv.host_fetch_bytes(l) for l in range(M)) - led0
        cold = {"ms": round(cold_ms, 3), "host_bytes": int(cold_bytes),
                "host_link_gbs": round(cold_bytes / (cold_ms / 1e3) / 1e9, 2)}

    # eager steps, then ONE CUDA graph of the step over the static input buffers
    for _ in range(n_eager):
        load(take())
        body()
    torch.cuda.synchronize()
    stream = torch.cuda.Stream(device=dev)
    graph = None
    try:
        with torch.cuda.stream(stream):
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                body()
        torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001 -- report and time the eager step instead
        print(f"[bench] CUDA graph capture failed ({type(e).__name__}: {e}); timing eager steps", file=sys.stderr)
        graph = None
        torch.cuda.synchronize()

    def run_step():
        load(take())
        if graph is not None:
            graph.replay()
        else:
            body()

    # warm-up: at least one replay (the graph's upload) before the timed region, whatever --warmup is
    for _ in range(max(1, args.warmup)):
        run_step()
    torch.cuda.synchronize()

    # ---------------- timed region: K steps (device time, CUDA events, max over ranks)
    ledger0 = sum(skv.host_fetch_bytes(l) for l in range(M)) if host else 0
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    cur = torch.cuda.current_stream()
    with ClockSampler(local) as clk:
        e0.record(cur)
        timed_k = []
        for k in range(args.steps):
            timed_k.append(nxt[0])
            load(take())
            ev[k][0].record(cur)
            if graph is not None:
                graph.replay()
            else:
                body()
            ev[k][1].record(cur)
        e1.record(cur)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_total = e0.elapsed_time(e1)
    step_ms = [a.elapsed_time(b) for a, b in ev]  # the replays alone (without the input copies)
    kern_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([ms_total, kern_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total, kern_ms = float(t[0].item()), float(t[1].item())
    ms_step = ms_total / args.steps
    value = GB / (ms_step / 1e3)
    host_step_bytes = (sum(skv.host_fetch_bytes(l) for l in range(M)) - ledger0) / args.steps if host else 0
    link_gbs = None
    if host:  # the host link's copy rate on this box (pinned -> HBM, 256 MB, CUDA events): the link roofline
        hsrc = torch.empty(1 << 28, dtype=torch.uint8).pin_memory()
        hdst = torch.empty(1 << 28, dtype=torch.uint8, device=dev)
        lk = []
        for _ in range(3):
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record()
            hdst.copy_(hsrc, non_blocking=True)
            b_.record()
            torch.cuda.synchronize()
            lk.append(a_.elapsed_time(b_))
        link_gbs = (1 << 28) / (min(lk) / 1e3) / 1e9
        del hsrc, hdst

    # ---------------- end-of-run check: one more step, eager, with its selections; sampled units
    # against the CPU oracle replaying this context's whole decode history (Eq. 2 state included)
    chk = None
    if check:
        ids_all = torch.empty((len(keep_layers), Bl, Gl, tau), dtype=torch.int32, device=dev)
        k_last = take()
        load(k_last)
        for l in range(M):
            skv.decode_step(l, qbuf[l], tbuf, outs[l], sel_ids=ids_all[l] if l < len(keep_layers) else None)
        torch.cuda.synchronize()
        chk = end_check(cfg, toks, Kh, Vh, keep_layers, history, qall, script, ids_all.cpu().numpy(),
                        outs.cpu().numpy(), Bl, Gl, Hl)

    # ---------------- per-kernel durations (profiled eager pass, events on the launching stream)
    # A spin kernel queued first lets the host enqueue the whole profiled pass ahead of the GPU,
    # so the events bracket back-to-back kernels rather than host launch gaps.
    skv.set_profiling(True)
    tok_hist = []
    torch.cuda.synchronize()
    torch.cuda._sleep(int(2e9 * 0.05))  # ~50 ms head start
    lc0 = skv.launch_count()
    for _ in range(n_prof):
        load(take())
        body(with_tokens=True)
        tok_hist.append(sel_tok.sum())
    torch.cuda.synchronize()
    launches_per_step = (skv.launch_count() - lc0) // n_prof
    ntok_sum = int(torch.stack(tok_hist).sum())
    prof = skv.profile_read()
    skv.set_profiling(False)
    S_tot = sum(S)
    unit_path = prof["step"][1] > 0  # one-launch step kernel; else the split kernels (Quest, skip fill)
    # algorithmic bytes per layer (this rank's Bl x Gl units); DESIGN.md section 9
    kv_bytes = ntok_sum * d * 2 * 2 / max(1, n_prof * M)        # selected K and V rows per layer
    e_bytes = Gl * S_tot * d * 2 * (2 if args.buckets == "quest" else 1)  # bf16 embeddings (Quest: min + max)
    qo_bytes = Bl * Hl * d * (2 + 4 + 4 + 4)                     # q, Sq read + write, O
    unit_bytes = e_bytes + kv_bytes + Gl * S_tot * 4 * 2 + qo_bytes  # + scores written, offsets read
    kern = {}
    name = "step" if unit_path else "split(score+select+attend)"
    iso = prof["step"] if unit_path else tuple(map(sum, zip(prof["score"], prof["select"], prof["attend"])))
    kern[name] = {"avg_us_isolated": round(iso[0] / max(1, n_prof * M) * 1e3, 3), "bytes_per_launch": int(unit_bytes)}
    # achieved: algorithmic bytes per layer / the layer's device time in the timed region = the graph
    # replays' device time (CUDA events on the replay stream, input copies excluded) / (steps x layers)
    launches_timed = M * args.steps
    avg_us = kern_ms * 1e3 / launches_timed
    kern[name]["avg_us"] = round(avg_us, 3)
    kern[name]["gbs"] = round(unit_bytes / (avg_us / 1e6) / 1e9, 1)
    kern[name]["share"] = round(kern_ms / ms_total, 4)
    traffic = None
    tf = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(tf) and plain:
        # dram__bytes_read.sum + dram__bytes_write.sum per launch of the step kernel, from one
        # `ncu --set full` capture of this workload and residency (scripts/gpu_profile.sh)
        with open(tf) as f:
            traffic = json.load(f).get(f"step_{residency}")
    roofline = {"bound": "hbm", "kernel": "unit_step_kernel (decode_unit.cu)" if unit_path else
                "score/quest_score + select (+ skip_fill) + attend_mma kernels per layer",
                "achieved": kern[name]["gbs"],
                "peak": hbm_peak, "unit": "GB/s", "frac": round(kern[name]["gbs"] / hbm_peak, 4),
                "traffic": traffic, "peak_kind": peak_kind,
                "duration": "graph replays' device time in the timed region / (steps x layers)",
                "per_unit": "per layer (all units): G*S*d*2 B (bf16 E; Quest pages: min + max) + sum(ntok)*d*2*2 B "
                            "(selected K,V rows) + G*S*4*2 (scores written, offsets read) + B*Hq*d*14 (q, Sq r/w, O)"}
    if host:  # the HBM fraction alone understates a step whose topic switches wait on PCIe
        roofline["note"] = ("host residency: part of the selected K/V comes over the host link (see "
                            "host_residency.link_roofline, the serial HBM + link bound)")

    # ---------------- the split call pair of SURVEY 8(b): decode_select + decode_attend per layer
    split = None
    if not args.no_split:
        torch.cuda.synchronize()
        sgraph = None
        try:
            load(take())
            body(split=True)  # eager (first split step: working-set path switch in host residency)
            torch.cuda.synchronize()
            with torch.cuda.stream(stream):
                sgraph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(sgraph, stream=stream):
                    body(split=True)
            torch.cuda.synchronize()
        except Exception as e:  # noqa: BLE001
            print(f"[bench] split-call graph capture failed ({e})", file=sys.stderr)
            sgraph = None
        n_sw = max(2, args.warmup)
        n_st = min(args.steps, 100)
        for _ in range(n_sw):
            load(take())
            sgraph.replay() if sgraph is not None else body(split=True)
        torch.cuda.synchronize()
        sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_st)]
        for k in range(n_st):
            load(take())
            sev[k][0].record(cur)
            sgraph.replay() if sgraph is not None else body(split=True)
            sev[k][1].record(cur)
        torch.cuda.synchronize()
        sms = [a.elapsed_time(b) for a, b in sev]
        sm = sum(sms) / n_st
        split = {"calls": "sentencekv_decode_select + sentencekv_decode_attend per layer (score, select, attend "
                          "kernels)", "steps": n_st, "ms_per_step": round(sm, 5), "value": round(GB / (sm / 1e3), 2),
                 "unit": "tokens/s", "p50_ms": round(pct(sms, 50), 5), "gpu_launches_per_step": 3 * M,
                 "cuda_graph": sgraph is not None}

    # ---------------- end to end through the public API with host buffers
    ne = args.e2e_steps
    k0 = nxt[0] % max(1, NQ - ne)
    qhost = qall[k0:k0 + ne].cpu().pin_memory()  # fresh queries per step, pinned host memory
    thost = tall[k0:k0 + ne].cpu().pin_memory()
    ohost = torch.empty((M, Bl, Hl, d), dtype=torch.float32).pin_memory()
    qdev = torch.empty((M, Bl, Hl, d), dtype=torch.bfloat16, device=dev)
    tdev = torch.empty((Bl,), dtype=torch.int32, device=dev)
    odev = torch.empty((M, Bl, Hl, d), dtype=torch.float32, device=dev)
    # each layer's output is read back on a copy stream as soon as its kernel is done, so the
    # device->host read of the step's result overlaps the later layers
    cstream = torch.cuda.Stream(device=dev)
    ev_o = [torch.cuda.Event() for _ in range(M)]

    def e2e_step(j):
        c = torch.cuda.current_stream()
        qdev.copy_(qhost[j], non_blocking=True)
        tdev.copy_(thost[j], non_blocking=True)
        for l in range(M):
            if kvbuf is not None:  # NEXT-2 (the step's K/V from the device pool, not counted in h2d)
                skvlib.sentencekv_decode_append(skv.ctx, l, kvall[k0 + j, l, 0], kvall[k0 + j, l, 1], tdev)
            skvlib.sentencekv_decode_step(skv.ctx, l, qdev[l], tdev, odev[l])
            if fused:
                skv.wait_outputs(l)
            elif world > 1:
                parallel.all_gather_outputs(odev[l], plan, gathered=gath[l])
            ev_o[l].record(c)
            with torch.cuda.stream(cstream):
                cstream.wait_event(ev_o[l])
                ohost[l].copy_(odev[l], non_blocking=True)
        c.synchronize()
        cstream.synchronize()

    for j in range(min(3, ne)):
        e2e_step(j)
    if world > 1:
        dist.barrier()
    x0 = torch.cuda.Event(enable_timing=True)
    x1 = torch.cuda.Event(enable_timing=True)
    x0.record()
    for j in range(ne):
        e2e_step(j)
    x1.record()
    torch.cuda.synchronize()
    e2e_ms = x0.elapsed_time(x1) / ne
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": round(GB / (e2e_ms / 1e3), 2), "unit": "tokens/s", "ms_per_step": round(e2e_ms, 4),
           "h2d_bytes_per_step": int(qhost[0].numel() * 2 + Bl * 4), "d2h_bytes_per_step": int(ohost.numel() * 4),
           "call": "sentencekv_decode_step per layer, eager from Python, fresh pinned-host queries each step"}

    # ---------------- CPU oracle baseline (rank 0, N=1 only; bounded sample of full steps)
    cpu = None
    if cpu_leg:
        ost = OracleStep(cfg | {"B": Bl}, toks, Kh, Vh)
        q_np = [qall[k].view(torch.int16).cpu().numpy().view(np.uint16) for k in range(4)]
        times = time_oracle(ost, q_np, script[:4], 30, budget_s=15.0)
        step_s = sum(times) / len(times)
        cpu = {"value": round(Bl / step_s, 4), "unit": "tokens/s", "cores": ost.threads, "kind": "oracle",
               "ms_per_step": round(step_s * 1e3, 1),
               "sample": f"{len(times)} full decode steps (all {M} layers x all {Bl * Gl} (b,g) units, select + "
                         f"attend, units in parallel on {ost.threads} threads); K/V bytes of layers "
                         f"{keep_layers} reused for the other layers (same shapes, same work)"}

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 5), "higher_is_better": True,
            "scaling": "weak" if args.shard == "batch" else "strong", "vs_baseline": None,
            "dtype": "bf16 in / fp32 acc (selection canonical fp32)",
            "data": "synthetic (seeded token streams with punctuation boundaries, topic-structured K/V/q; fresh "
                    "queries every step, topic switch after each boundary input)",
            "config": config_dict(args, cfg, GB),
            "run": {"sentences_rank0": S, "residency": "pinned host K/V + HBM working set" if host else "device (HBM)",
                    "parallelism": f"{plan.batch_shards} batch x {plan.head_shards} KV-head shards"
                                   + (", fused gather epilogue" if fused else (", NCCL all-gather" if world > 1 else "")),
                    "l2": f"inputs > L2: {(e_bytes + kv_bytes) * M / 1e9:.2f} GB read per step per GPU (L2 126 MB), "
                          "no flush needed",
                    "cuda_graph": graph is not None},
            # boundary inputs (-> Q_s reset, new query topic) among the timed steps' inputs: in host residency
            # each one brings that sequence's newly selected sentences over PCIe, so short runs vary with it
            "boundary_inputs_timed": int(np.isin(script[timed_k], synth.BOUNDARY_IDS).sum()),
            "step_ms": {"p10": round(pct(step_ms, 10), 5), "p50": round(pct(step_ms, 50), 5),
                        "p90": round(pct(step_ms, 90), 5), "max": round(max(step_ms), 5),
                        "note": "per-step graph replay device time (input copy excluded)"},
            "roofline": roofline,
            "kernels": kern,
            "e2e": e2e,
            "split_calls": split,
            # kernels of this library per timed step: one unit_step_kernel per layer (decode_unit.cu)
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "prefill": {"ms": round(prefill_ms, 3), "K_bytes": int(Bl * Gl * L * d * 2 * M),
                        "segment_ms": round(prof_prefill["segment"][0], 3),
                        "compress_ms_per_layer": round(prof_prefill["compress"][0] / max(1, prof_prefill["compress"][1]), 4),
                        "compress_gbs": round(Bl * Gl * (skv.retained_tokens(0) if N else L) * d * 2 / (prof_prefill["compress"][0] / max(1, prof_prefill["compress"][1]) / 1e3) / 1e9, 1)},
            "host_residency": {"host_bytes_per_step": int(host_step_bytes),
                               "host_rows_per_step": round(host_step_bytes / (d * 2 * 2), 1),
                               "host_link_gbs_in_step": round(host_step_bytes / (ms_step / 1e3) / 1e9, 2),
                               # P3: D2H copy time on the copy stream (CUDA events)
                               "offload_gbs_p3": round(kv_bytes_total / (prof_prefill["offload"][0] / 1e3) / 1e9, 2)
                               if prof_prefill["offload"][1] else None,
                               "offload_wall_s_incl_pinning": round(offload_s, 2) if offload_s else None,
                               "page_cache_tokens_per_unit": int(2.0 * tau), "cold_first_step": cold,
                               "paper_onload": "PAPER.md P:740: onload 1024 tokens 0.0038 s (H100 NVL, per step)",
                               # host residency is bound by HBM AND the host link, one after the other
                               # (the rows to fetch are known only after the selection): the step's
                               # lower bound is HBM bytes / HBM peak + host bytes / link copy rate
                               "link_roofline": {
                                   "bound": "hbm + host link (serial)", "link_gbs_measured": round(link_gbs, 2),
                                   "hbm_bytes_per_step": int(unit_bytes * M), "host_bytes_per_step": int(host_step_bytes),
                                   "t_min_ms": round((unit_bytes * M / (hbm_peak * 1e9) + host_step_bytes / (link_gbs * 1e9)) * 1e3, 4),
                                   "frac": round((unit_bytes * M / (hbm_peak * 1e9) + host_step_bytes / (link_gbs * 1e9)) * 1e3 / ms_step, 4)}}
            if host else None,
            "end_check": chk,
            "retention": ret,
            "cpu_baseline": cpu,
            "kv_gen_s": round(t_gen, 2),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def end_check(cfg, toks, Kh, Vh, layers, history, qall, script, ids_g, O_g, Bl, Gl, Hl):
    """CHECK_UNITS sampled (layer, b, g) units of the last executed step against the CPU oracle: the
    oracle replays the Eq. 2 query cache of the unit's (layer, b) over the whole decode history of
    the context, then scores, selects and attends at the last step.  ids bit-exact, O <= 2e-3."""
    import oracle
    import synth

    tau, grp, d = cfg["tau"], cfg["Hq"] // cfg["G"], cfg["d"]
    rng = np.random.default_rng(17)
    units = sorted({(int(rng.integers(len(layers))), int(rng.integers(Bl)), int(rng.integers(Gl)))
                    for _ in range(CHECK_UNITS)})
    bset = set(synth.BOUNDARY_IDS.tolist())
    worst, ok = 0.0, True
    for li, b, g in units:
        l = layers[li]
        off = oracle.segment(toks[b], synth.BOUNDARY_IDS, tau)
        E = oracle.embed(Kh[li][b, g], off)
        Sq = np.zeros((Hl, d), np.float32)
        cnt = np.zeros(1, np.int32)
        qs = qall[history, l, b].view(__import__("torch").int16).cpu().numpy().view(np.uint16)  # [steps][Hl][d]
        for j, k in enumerate(history):
            qbar = oracle.qs_append_mean(Sq, cnt, qs[j])
            if j + 1 < len(history) and int(script[k][b]) in bset:
                oracle.qs_reset(Sq, cnt)
        sc = oracle.score(oracle.group_query(qbar, grp, g), E)
        ids, _ = oracle.select(sc, off, tau)
        n = len(ids)
        same = bool(np.array_equal(ids_g[li, b, g, :n], ids) and np.all(ids_g[li, b, g, n:] == -1))
        O = oracle.attend(qs[-1][g * grp:(g + 1) * grp], Kh[li][b, g], Vh[li][b, g], off, ids)
        err = float(np.max(np.abs(O_g[l, b, g * grp:(g + 1) * grp] - O)))
        worst = max(worst, err)
        ok = ok and same and err <= 2e-3
    return {"units": [list(u) for u in units], "steps_replayed": len(history), "ids_bit_exact_and_O_2e-3": ok,
            "max_abs_O": worst}


def reference_arm(args, cfg, rank, world, residency):
    """--impl reference: the CPU oracle as it stands (oracle/), on this arm's config, metric and unit.
    Each step is one FULL decode step (all layers x all (b, g) units, select + attend, units in
    parallel on every host thread).  Host RAM holds one layer of K/V, so every layer reuses its
    bytes (same shapes, same work).  Rank 0 only; other ranks exit without work."""
    if rank != 0:
        return
    import synth

    B, M, Hq, G, d, L, tau = (cfg[k] for k in ("B", "M", "Hq", "G", "d", "L", "tau"))
    GB = B * world if args.shard == "batch" else B
    toks, topics = synth.prompts(SEED, GB, L, cfg["median"])
    K, V = synth.kv_layer(SEED, 0, topics, G, d)
    ost = OracleStep(cfg | {"B": GB}, toks, [K], [V])
    script, target = synth.decode_script(SEED, GB, 8)
    qsteps = [[synth.queries(SEED, l, s, target[s], Hq, G, d) for l in range(M)] for s in range(8)]
    time_oracle(ost, qsteps, script, max(1, args.warmup))
    times = time_oracle(ost, qsteps, script, args.steps)
    step_s = sum(times) / len(times)
    value = GB / step_s
    cpu = {"value": round(value, 4), "unit": "tokens/s", "cores": ost.threads, "kind": "oracle",
           "sample": f"{len(times)} full decode steps (all {M} layers x all {GB * G} (b,g) units, select + attend); "
                     f"one layer's K/V bytes reused by every layer (host RAM)"}
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_s * 1e3, 3),
            "higher_is_better": True, "scaling": "weak" if args.shard == "batch" else "strong",
            "vs_baseline": None, "dtype": "fp32 canonical selection / fp64 attention", "data": "synthetic",
            "config": config_dict(args, cfg, GB),
            "run": {"residency": "host RAM (oracle)", "parallelism": f"{ost.threads} CPU threads"},
            "cpu_baseline": cpu,
            "e2e": {"value": round(value, 4), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
