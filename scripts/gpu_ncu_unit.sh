#!/bin/bash
# ncu: full capture of one unit_step_kernel launch (device residency, 8b-128k), plus launch list
mkdir -p gpurun_out
tag=${1:-unit}
shift
env "$@" timeout 900 ncu --set full --clock-control none --import-source on -k regex:unit_step -s 40 -c 1 \
   -o gpurun_out/prof_$tag python bench.py --steps 2 --warmup 1 --residency device --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_$tag.log 2>&1
tail -3 gpurun_out/ncu_$tag.log
env "$@" timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"unit_step|score|select|attend" -c 200 --csv \
   --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 1 --residency device --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
ls -la gpurun_out | tail -5
