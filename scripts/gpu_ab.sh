#!/bin/bash
# A/B bench: PDL on vs off, plus GPU tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --steps 300 --warmup 10 > gpurun_out/bench_128k.txt 2>&1
SKV_PDL=1 timeout 900 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/bench_128k_pdl.txt 2>&1
python - <<'PY'
import json
for f in ["gpurun_out/bench_128k.txt", "gpurun_out/bench_128k_pdl.txt"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], d["step_gbs"], {k: v["avg_us"] for k, v in d["kernels"].items()}, d["e2e"]["ms_per_step"])
    except Exception as e:
        print(f, "ERR", e, open(f).read()[-2000:])
PY
