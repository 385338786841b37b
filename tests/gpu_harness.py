"""Shared driver for the GPU parity tests: runs the CUDA path through the C ABI (python binding)
and the CPU oracle on the same seeded inputs, step by step, and compares."""
from __future__ import annotations

import numpy as np
import torch

import oracle
import synth

ATOL = 2e-3  # north_star: max-abs 2e-3 for bf16 inputs with fp32 accumulation


def to_bits(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def from_bits(a: np.ndarray, device) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).to(device).view(torch.bfloat16)


def run_parity(skv, orc: oracle.Oracle, toks, Ks, Vs, qs, script_tok, bset, device, check_scores=True,
               units=None, mode="split"):
    """Prefill all layers, then decode len(qs) steps over all layers, comparing every step.

    Ks/Vs: per layer bf16 bits [B][G][L][d]; qs[step][layer]: bf16 bits [B][Hq][d].
    units: optional list of (b, g) to compare (default: all).
    mode: "split" = sentencekv_decode_select + sentencekv_decode_attend; "step" =
    sentencekv_decode_step (fused select + attend); "graph" = as bench.py times it: step 0 eager,
    then ONE CUDA graph of sentencekv_decode_step over all layers, captured once over static input
    buffers and replayed for every later step with that step's inputs copied in.
    Returns a dict of statistics."""
    B, G, tau = skv.B, skv.G, skv.tau
    M = len(Ks)
    tok_dev = torch.from_numpy(np.ascontiguousarray(toks)).to(device)
    Kd = [from_bits(K, device) for K in Ks]
    Vd = [from_bits(V, device) for V in Vs]
    for l in range(M):
        skv.prefill_compress(l, Kd[l], Vd[l], token_ids=tok_dev if l == 0 else None,
                             boundary_ids=bset if l == 0 else None)
        orc.prefill_layer(l, Ks[l], Vs[l])
    torch.cuda.synchronize()
    units = units or [(b, g) for b in range(B) for g in range(G)]
    stats = {"max_abs": 0.0, "steps": 0, "sel_tokens": []}

    # P1: offsets bit-exact
    S = skv.sentence_counts()
    off = skv.offsets().cpu().numpy()
    for b in range(B):
        assert S[b] == len(orc.off[b]) - 1, f"S[{b}]"
        assert np.array_equal(off[b, : S[b] + 1], orc.off[b]), f"offsets b={b}"
    # P2: E bit-exact
    for l in range(M):
        E = to_bits(skv.embeddings(l))
        for b, g in units:
            assert np.array_equal(E[b, g, : S[b]], orc.E[l][b][g]), f"E l={l} b={b} g={g}"

    sel_ids = torch.empty((B, G, tau), dtype=torch.int32, device=device)
    sel_cnt = torch.empty((B, G), dtype=torch.int32, device=device)
    sel_tok = torch.empty((B, G), dtype=torch.int32, device=device)
    out = torch.empty((B, skv.Hq, skv.d), dtype=torch.float32, device=device)
    graph = None
    if mode == "graph":  # static buffers of the captured step, one set of outputs per layer
        gq = [torch.empty((B, skv.Hq, skv.d), dtype=torch.bfloat16, device=device) for _ in range(M)]
        git = torch.empty((B,), dtype=torch.int32, device=device)
        gids = [torch.empty_like(sel_ids) for _ in range(M)]
        gcnt = [torch.empty_like(sel_cnt) for _ in range(M)]
        gtok = [torch.empty_like(sel_tok) for _ in range(M)]
        gout = [torch.empty_like(out) for _ in range(M)]
    for step, qstep in enumerate(qs):
        it = torch.from_numpy(np.ascontiguousarray(script_tok[step])).to(device)
        if mode == "graph" and step > 0:
            for l in range(M):
                gq[l].copy_(from_bits(qstep[l], device))
            git.copy_(it)
            if graph is None:
                torch.cuda.synchronize()
                cs = torch.cuda.Stream(device=device)
                with torch.cuda.stream(cs):
                    graph = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(graph, stream=cs):
                        for l in range(M):
                            skv.decode_step(l, gq[l], git, gout[l], gids[l], gcnt[l], gtok[l])
                torch.cuda.synchronize()
            graph.replay()
            torch.cuda.synchronize()
        for l in range(M):
            q_bits = qstep[l]
            qd = from_bits(q_bits, device)
            if mode == "graph" and step > 0:
                pass  # this step already ran (graph replay)
            elif mode in ("step", "graph"):
                skv.decode_step(l, qd, it, out, sel_ids, sel_cnt, sel_tok)
            else:
                skv.decode_select(l, qd, it, sel_ids, sel_cnt, sel_tok)
                skv.decode_attend(l, qd, out)
            sc_o, ids_o, ntok_o = orc.decode_select(l, q_bits, script_tok[step])
            O_o = orc.decode_attend(l, q_bits, ids_o)
            replayed = mode == "graph" and step > 0
            ids_g = (gids[l] if replayed else sel_ids).cpu().numpy()
            cnt_g = (gcnt[l] if replayed else sel_cnt).cpu().numpy()
            tok_g = (gtok[l] if replayed else sel_tok).cpu().numpy()
            O_g = (gout[l] if replayed else out).cpu().numpy()
            sc_g = skv.scores(l).cpu().numpy() if check_scores else None
            for b, g in units:
                if check_scores:
                    assert np.array_equal(sc_g[b, g, : S[b]].view(np.uint32), sc_o[b][g].view(np.uint32)), \
                        f"scores step={step} l={l} b={b} g={g}"
                n = len(ids_o[b][g])
                assert cnt_g[b, g] == n, f"count step={step} l={l} b={b} g={g}: {cnt_g[b, g]} vs {n}"
                assert np.array_equal(ids_g[b, g, :n], ids_o[b][g]), f"ids step={step} l={l} b={b} g={g}"
                assert np.all(ids_g[b, g, n:] == -1)
                assert tok_g[b, g] == ntok_o[b][g] <= tau
                hs = slice(g * skv.grp, (g + 1) * skv.grp)
                err = float(np.max(np.abs(O_g[b, hs] - O_o[b, hs])))
                stats["max_abs"] = max(stats["max_abs"], err)
                stats["sel_tokens"].append(int(tok_g[b, g]))
                assert err <= ATOL, f"O step={step} l={l} b={b} g={g}: {err}"
        stats["steps"] += 1
    return stats


def make_case(seed, B, M, Hq, G, d, L, tau, steps, median):
    toks, topics = synth.prompts(seed, B, L, median=median)
    Ks, Vs = zip(*(synth.kv_layer(seed, l, topics, G, d) for l in range(M)))
    script_tok, target = synth.decode_script(seed, B, steps)
    qs = [[synth.queries(seed, l, s, target[s], Hq, G, d) for l in range(M)] for s in range(steps)]
    return toks, topics, list(Ks), list(Vs), qs, script_tok
