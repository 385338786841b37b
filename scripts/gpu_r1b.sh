#!/bin/bash
# GPU call: parity tests, bench (8b-128k), ncu launch list + full captures of the decode kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --steps 300 --warmup 10 > gpurun_out/bench_128k.txt 2>&1
tail -c 3000 gpurun_out/bench_128k.txt
if [ "$1" == "ncu" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"segment|compress|score|select|attend" -c 400 --csv \
     --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
  for k in attend_kernel score_kernel select_kernel; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 20 -c 1 \
       -o gpurun_out/prof_$k python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_$k.log 2>&1
  done
  ls -la gpurun_out
fi
