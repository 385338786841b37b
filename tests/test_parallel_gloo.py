"""Multi-GPU host logic on CPU: shard planning, the per-layer all-gather of per-head
outputs and its assembly, run with world_size 2 over gloo; plus a shard simulation of the whole
decode step with the CPU oracle (each rank computes its own units, the gathered result must equal
the single-process result -- selection is shard-local)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_00970_b200 import parallel


@pytest.mark.parametrize("B,G,Hq,world,strategy", [
    (4, 8, 32, 1, "heads"), (4, 8, 32, 2, "heads"), (4, 8, 32, 4, "heads"), (4, 8, 32, 8, "heads"),
    (16, 8, 64, 8, "heads"), (16, 8, 64, 8, "batch"), (1, 8, 32, 8, "heads"), (4, 2, 8, 8, "heads"),
    (8, 4, 16, 2, "batch"),
])
def test_plan_covers_every_unit_once(B, G, Hq, world, strategy):
    owner = {}
    for r in range(world):
        p = parallel.plan(B, G, Hq, world, r, strategy)
        assert p.batch_count * p.batch_shards == B and p.kv_head_count * p.head_shards == G
        for b in range(p.batch_begin, p.batch_begin + p.batch_count):
            for g in range(p.kv_head_begin, p.kv_head_begin + p.kv_head_count):
                assert (b, g) not in owner
                owner[(b, g)] = r
        assert p.q_head_begin == p.kv_head_begin * (Hq // G) and p.q_head_count == p.kv_head_count * (Hq // G)
    assert len(owner) == B * G


def test_plan_rejects_uneven_splits():
    with pytest.raises(ValueError):
        parallel.plan(3, 8, 32, 16, 0, "heads")  # 8 head shards x 2 batch shards: B=3 not divisible


def test_assemble_single_rank_identity():
    p = parallel.plan(2, 4, 8, 1, 0)
    x = torch.randn(1, 2, 8, 16)
    assert torch.equal(parallel.assemble(x, p), x[0])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # surfaced by the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _spawn(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    return res


def _gather_fn(rank, world):
    B, G, Hq, d = 4, 4, 16, 8
    ok = []
    for strategy in ("heads", "batch"):
        p = parallel.plan(B, G, Hq, world, rank, strategy)
        full = torch.arange(B * Hq * d, dtype=torch.float32).view(B, Hq, d)
        local = full[p.batch_begin:p.batch_begin + p.batch_count,
                     p.q_head_begin:p.q_head_begin + p.q_head_count].contiguous()
        got = parallel.assemble(parallel.all_gather_outputs(local, p), p)
        ok.append(bool(torch.equal(got, full)))
    return ok


def test_all_gather_assembles_heads_and_batch_gloo_ws2():
    res = _spawn(_gather_fn)
    assert res == {0: [True, True], 1: [True, True]}, res


def _shard_sim_fn(rank, world):
    """Each rank runs the oracle decode step on its units only; the gathered outputs and selections
    must equal a single-process oracle run over all units."""
    import oracle
    import synth

    B, M, Hq, G, d, L, tau, steps = 2, 1, 8, 2, 64, 2048, 128, 4
    toks, topics = synth.prompts(5, B, L, median=20.0)
    K, V = synth.kv_layer(5, 0, topics, G, d)
    script, target = synth.decode_script(5, B, steps)
    p = parallel.plan(B, G, Hq, world, rank, "heads")
    bs = slice(p.batch_begin, p.batch_begin + p.batch_count)
    gs = slice(p.kv_head_begin, p.kv_head_begin + p.kv_head_count)
    hs = slice(p.q_head_begin, p.q_head_begin + p.q_head_count)
    local = oracle.Oracle(toks[bs], synth.BOUNDARY_IDS, tau, M, p.q_head_count, p.kv_head_count, d)
    local.prefill_layer(0, K[bs, gs], V[bs, gs])
    full = oracle.Oracle(toks, synth.BOUNDARY_IDS, tau, M, Hq, G, d)
    full.prefill_layer(0, K, V)
    ok = True
    for s in range(steps):
        q = synth.queries(5, 0, s, target[s], Hq, G, d)
        _, ids_l, _ = local.decode_select(0, q[bs, hs], script[s, bs])
        O_l = torch.from_numpy(local.decode_attend(0, q[bs, hs], ids_l).astype(np.float32))
        _, ids_f, _ = full.decode_select(0, q, script[s])
        O_f = torch.from_numpy(full.decode_attend(0, q, ids_f).astype(np.float32))
        got = parallel.assemble(parallel.all_gather_outputs(O_l, p), p)
        ok &= bool(torch.equal(got, O_f))
        for bi in range(p.batch_count):
            for gi in range(p.kv_head_count):
                ok &= np.array_equal(ids_l[bi][gi], ids_f[p.batch_begin + bi][p.kv_head_begin + gi])
    return ok


def test_shard_simulation_of_decode_step_gloo_ws2():
    res = _spawn(_shard_sim_fn)
    assert res == {0: True, 1: True}, res
