#!/bin/bash
# r02 evidence set: GPU tests, smoke, the default bench (driver-style and long), device residency,
# reference arm, configs[1]/[3], the NEXT-row lines.  Outputs in gpurun_out/$TAG.
O=gpurun_out/${TAG:-final}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout -s KILL 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 > $O/bench_host_short.txt 2>&1; tail -c 200 $O/bench_host_short.txt; echo
timeout -s KILL 900 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > $O/bench_host_long.txt 2>&1; tail -c 200 $O/bench_host_long.txt; echo
timeout -s KILL 900 python bench.py --residency device --steps 300 --warmup 10 --no-cpu-baseline > $O/bench_dev_long.txt 2>&1; tail -c 200 $O/bench_dev_long.txt; echo
timeout -s KILL 900 python bench.py --residency device --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_dev_short.txt 2>&1; tail -c 200 $O/bench_dev_short.txt; echo
timeout -s KILL 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.txt 2>&1; tail -c 200 $O/bench_ref.txt; echo
TAG=$TAG/cfg bash scripts/gpu_configs.sh
TAG=$TAG/vb bash scripts/gpu_variants_bench.sh
timeout -s KILL 600 python bench.py --local --residency device --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 10 > $O/bench_local.txt 2>&1; tail -c 200 $O/bench_local.txt; echo
