#!/bin/bash
# GPU call: parity tests, smoke, bench (device + host residency), ncu launch list + full captures
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 600 python bench.py --steps 300 --warmup 10 --residency device --no-cpu-baseline > gpurun_out/bench_dev.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_host.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.txt 2>&1
python - <<'PY'
import json
for f in ["gpurun_out/bench_dev.txt", "gpurun_out/bench_host.txt", "gpurun_out/bench_ref.txt"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], {k: v["avg_us"] for k, v in d.get("kernels", {}).items()}, d["e2e"], d.get("roofline"), d.get("cpu_baseline"))
    except Exception as e:
        print(f, "ERR", e, open(f).read()[-2000:])
PY
if [ "$1" == "ncu" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"segment|compress|score|select|attend|layer" -c 400 --csv \
     --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
  for k in attend_mma score_kernel select_kernel; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 20 -c 1 \
       -o gpurun_out/prof_$k python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_$k.log 2>&1
  done
  ls -la gpurun_out
fi
