#!/bin/bash
# r02 (last session) evidence set: GPU tests, smoke, the default bench (driver-style and long), device
# residency, reference arm, configs[1]/[3], NEXT-row lines (NEXT-2 in both residencies), ncu launch
# lists + full captures of the step kernel, compute-sanitizer.  Outputs in gpurun_out/$TAG.
TAG=${TAG:-final_b}; O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout -s KILL 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 > $O/bench_host_short.txt 2>&1; tail -c 150 $O/bench_host_short.txt; echo
timeout -s KILL 900 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > $O/bench_host_long.txt 2>&1; tail -c 150 $O/bench_host_long.txt; echo
timeout -s KILL 900 python bench.py --residency device --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_dev_short.txt 2>&1; tail -c 150 $O/bench_dev_short.txt; echo
timeout -s KILL 900 python bench.py --residency device --steps 300 --warmup 10 --no-cpu-baseline > $O/bench_dev_long.txt 2>&1; tail -c 150 $O/bench_dev_long.txt; echo
timeout -s KILL 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.txt 2>&1; tail -c 150 $O/bench_ref.txt; echo
TAG=$TAG/cfg bash scripts/gpu_configs.sh
TAG=$TAG/vb bash scripts/gpu_variants_bench.sh
timeout -s KILL 600 python bench.py --local --residency device --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 10 > $O/bench_local_dev.txt 2>&1; tail -c 150 $O/bench_local_dev.txt; echo
timeout -s KILL 900 python bench.py --local --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 10 > $O/bench_local_host.txt 2>&1; tail -c 150 $O/bench_local_host.txt; echo
timeout -s KILL 600 python bench.py --local --retention --residency device --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 10 > $O/bench_retention_local.txt 2>&1; tail -c 150 $O/bench_retention_local.txt; echo
A="--steps 2 --warmup 1 --no-cpu-baseline --no-split --no-check --e2e-steps 1"
for res in device host; do
  timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
     -k regex:"segment|compress|unit_step|score|select|attend" -c 200 --csv --log-file $O/launches_$res.csv \
     python bench.py --residency $res $A > /dev/null 2>&1; echo "launches $res rc=$?"
  [ -n "$NO_FULL" ] || timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:unit_step -s 40 -c 1 \
     -o $O/prof_step_$res python bench.py --residency $res $A > $O/ncu_step_$res.log 2>&1; echo "full $res rc=$?"
done
TAG=$TAG/san bash scripts/gpu_sanitize.sh
ls $O
