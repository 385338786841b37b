#!/bin/bash
# first GPU call: tests, smoke, bench (tiny + 8b-128k), launch list
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py --config tiny --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_tiny.txt 2>&1
timeout 900 python bench.py --steps 200 --warmup 10 > gpurun_out/bench_128k.txt 2>&1
tail -5 gpurun_out/pytest_gpu.txt gpurun_out/smoke.txt gpurun_out/bench_tiny.txt gpurun_out/bench_128k.txt
