#!/bin/bash
# Round profile pass: GPU tests, benches (default = host residency with CPU baseline; device
# residency; reference arm), ncu launch lists of both residencies and one `ncu --set full` capture
# of the step kernel per residency.  Outputs under gpurun_out/ (copied to profiles/ by hand).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench_host.txt 2>&1; tail -c 300 gpurun_out/bench_host.txt; echo
timeout 600 python bench.py --residency device --no-cpu-baseline > gpurun_out/bench_dev.txt 2>&1; tail -c 300 gpurun_out/bench_dev.txt; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.txt 2>&1; tail -c 300 gpurun_out/bench_ref.txt; echo
for res in device host; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"segment|compress|unit_step|score|select|attend" -c 200 --csv \
     --log-file gpurun_out/launches_$res.csv python bench.py --steps 2 --warmup 1 --residency $res --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:unit_step -s 40 -c 1 \
     -o gpurun_out/prof_step_$res python bench.py --steps 2 --warmup 1 --residency $res --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_step_$res.log 2>&1
done
ls gpurun_out
