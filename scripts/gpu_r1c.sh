#!/bin/bash
# GPU call: parity tests, bench (device + host residency), phase trace, optional ncu captures
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 300 --warmup 10 --residency device --no-cpu-baseline > gpurun_out/bench_dev.txt 2>&1
timeout 900 python bench.py --steps 300 --warmup 10 > gpurun_out/bench_host.txt 2>&1
python - <<'PY'
import json
for f in ["gpurun_out/bench_dev.txt", "gpurun_out/bench_host.txt"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], d.get("step_gbs_per_gpu"), {k: v["avg_us"] for k, v in d["kernels"].items()}, d["e2e"]["ms_per_step"], d["roofline"])
    except Exception as e:
        print(f, "ERR", e, open(f).read()[-2000:])
PY
timeout 600 python scripts/trace_step.py > gpurun_out/trace.txt 2>&1; tail -25 gpurun_out/trace.txt
if [ "$1" == "ncu" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"segment|compress|score|select|attend" -c 400 --csv \
     --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
  for k in attend_mma score_kernel select_kernel; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 20 -c 1 \
       -o gpurun_out/prof_$k python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_$k.log 2>&1
  done
  ls -la gpurun_out
fi
