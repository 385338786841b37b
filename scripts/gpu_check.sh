#!/bin/bash
# GPU check of the current tree: parity tests, smoke, bench lines (driver-style short run and a long run,
# both residencies, the reference arm). Outputs under gpurun_out/$TAG.
TAG=${TAG:-check}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_host_short.txt 2>&1; tail -c 600 $O/bench_host_short.txt; echo
timeout 900 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > $O/bench_host_long.txt 2>&1; tail -c 300 $O/bench_host_long.txt; echo
timeout 600 python bench.py --residency device --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_dev.txt 2>&1; tail -c 300 $O/bench_dev.txt; echo
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.txt 2>&1; tail -c 300 $O/bench_ref.txt; echo
