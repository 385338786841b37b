#!/bin/bash
# Bench lines only: driver-style short run and a long run (host residency, configs[2]), device residency.
TAG=${TAG:-bench}
O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_host_short.txt 2>&1; tail -c 300 $O/bench_host_short.txt; echo
timeout 900 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > $O/bench_host_long.txt 2>&1; tail -c 300 $O/bench_host_long.txt; echo
timeout 600 python bench.py --residency device --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_dev.txt 2>&1; tail -c 300 $O/bench_dev.txt; echo
