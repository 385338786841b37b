#!/bin/bash
# quick iteration check: GPU tests, driver-style host + device bench lines (no CPU baseline)
TAG=${TAG:-quick}
O=gpurun_out/$TAG; mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_host_short.txt 2>&1
timeout 600 python bench.py --residency device --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_dev.txt 2>&1
for f in $O/bench_*.txt; do echo $f; tail -1 $f | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d.get('value'), d.get('ms_per_step'), d.get('step_ms'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('ms_per_step'))"; done
