"""bench.py's reference arm (the CPU oracle) runs without a GPU: its JSON line
must carry the contract's keys, and under torchrun only rank 0 prints it."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lines(out):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def test_reference_arm_json_contract():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "tiny", "--steps", "2",
                        "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    (line,) = _lines(r.stdout)
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["n_gpus"] == 1 and line["steps"] == 2 and line["warmup"] == 1
    assert line["config"]["workload"] == "tiny"
    assert line["value"] > 0 and line["higher_is_better"] is True
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    e = line["e2e"]
    assert e["value"] == line["value"] and e["unit"] == line["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_reference_arm_torchrun_rank0_only():
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29531", "bench.py", "--impl", "reference",
                        "--config", "tiny", "--gpus", "2", "--steps", "1", "--warmup", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    (line,) = _lines(r.stdout)
    assert line["impl"] == "reference" and line["n_gpus"] == 2


@pytest.mark.gpu
def test_bench_two_ranks_same_gpu():
    """The N > 1 path of bench.py (per-rank head shards, per-layer all-gather of the outputs,
    barriers, max over ranks, one line from rank 0) on ONE GPU: both ranks on cuda:0 with the gloo
    backend (SKV_BENCH_SAME_GPU=1; a test hook, not a measurement)."""
    env = dict(os.environ, SKV_BENCH_SAME_GPU="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29537", "bench.py", "--gpus", "2",
                        "--config", "8b-32k", "--residency", "device", "--steps", "4", "--warmup", "3",
                        "--e2e-steps", "2", "--no-cpu-baseline"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    (line,) = _lines(r.stdout)
    assert line["n_gpus"] == 2 and line["run"]["parallelism"].startswith("1 batch x 2 KV-head shards")
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] == 32 * 4
