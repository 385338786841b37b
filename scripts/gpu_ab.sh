#!/bin/bash
# A/B bench of step-kernel variants (device residency unless the name starts with "host").
# usage: scripts/gpu_ab.sh [tests] name[:ENV=V[,ENV=V]] ...
#   e.g. scripts/gpu_ab.sh tests base pf0:SKV_PF_NEXT=0 host hostpf0:SKV_PF_NEXT=0
mkdir -p gpurun_out
if [ "$1" == "tests" ]; then
  shift
  timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
fi
for spec in "$@"; do
  name=${spec%%:*}
  envs=""
  [ "$spec" != "$name" ] && envs=$(echo "${spec#*:}" | tr ',' ' ')
  res=device
  [[ $name == host* ]] && res=host
  env $envs timeout 600 python bench.py --steps 300 --warmup 10 --residency $res --no-cpu-baseline --e2e-steps 20 \
      > gpurun_out/bench_$name.txt 2>&1
  python - "$name" <<'PY'
import json, sys
f = f"gpurun_out/bench_{sys.argv[1]}.txt"
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(sys.argv[1], "ms/step", d["ms_per_step"], {k: (v["avg_us"], v["gbs"]) for k, v in d["kernels"].items()},
          "e2e", d["e2e"]["ms_per_step"], "frac", d["roofline"]["frac"], "clk", d["clocks"]["sm_mhz"])
except Exception as e:
    print(f, "ERR", e, open(f).read()[-1500:])
PY
done
