#!/bin/bash
# Round-end check: GPU tests, smoke, bench lines (default host residency with the CPU baseline,
# device residency, reference arm)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench_host.txt 2>&1; tail -c 400 gpurun_out/bench_host.txt; echo
timeout 600 python bench.py --residency device --no-cpu-baseline > gpurun_out/bench_dev.txt 2>&1; tail -c 400 gpurun_out/bench_dev.txt; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.txt 2>&1; tail -c 300 gpurun_out/bench_ref.txt; echo
