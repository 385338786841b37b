#!/bin/bash
# GPU call: parity tests, unit-kernel trace, A/B benches of decode_step variants (device residency)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python scripts/trace_unit.py > gpurun_out/trace_unit.txt 2>&1; tail -28 gpurun_out/trace_unit.txt
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 600 python bench.py --steps 300 --warmup 10 --residency device --no-cpu-baseline --e2e-steps 20 > gpurun_out/bench_$name.txt 2>&1
  python - "$name" <<'PY'
import json, sys
f = f"gpurun_out/bench_{sys.argv[1]}.txt"
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(sys.argv[1], "ms/step", d["ms_per_step"], {k: (v["avg_us"], v["gbs"]) for k, v in d["kernels"].items()}, "e2e", d["e2e"]["ms_per_step"], "frac", d["roofline"]["frac"])
except Exception as e:
    print(f, "ERR", e, open(f).read()[-1500:])
PY
}
for v in "$@"; do
  case $v in
    unit) run unit ;;
    nopf) run unit_nopf SKV_PREFETCH=0 ;;
    pdl) run unit_pdl SKV_PDL=1 ;;
    nopdl) run unit_nopdl SKV_PDL=0 ;;
    pull) run unit_pull SKV_PUSH_MERGE=0 ;;
    unit2) run unit2 ;;
    pull2) run unit_pull2 SKV_PUSH_MERGE=0 ;;
    prev) run prev SKV_LIB=paper_2504_00970_b200/libsentencekv_prev.so ;;
    prev2) run prev2 SKV_LIB=paper_2504_00970_b200/libsentencekv_prev.so ;;
    band0) run unit_band0 SKV_BAND_LOG2=0 ;;
    band21) run unit_band21 SKV_BAND_LOG2=21 ;;
    band17) run unit_band17 SKV_BAND_LOG2=17 ;;
    split) run split SKV_UNIT=0 ;;
  esac
done
for v in "$@"; do
  case $v in
    host)
      timeout 900 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 20 > gpurun_out/bench_host.txt 2>&1
      python - <<'PY'
import json
f = "gpurun_out/bench_host.txt"
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print("host ms/step", d["ms_per_step"], {k: (v["avg_us"], v["gbs"]) for k, v in d["kernels"].items()}, "e2e", d["e2e"]["ms_per_step"], "frac", d["roofline"]["frac"], d.get("host_residency"))
except Exception as e:
    print(f, "ERR", e, open(f).read()[-1500:])
PY
      ;;
  esac
done
