#!/bin/bash
# r02 ncu evidence: launch lists (device / host residency) of the default bench workload, one full
# capture of the step kernel per residency, one full capture of the NEXT-1 tcgen05 kernels.
O=gpurun_out/${TAG:-ncu2}; mkdir -p $O
A="--steps 2 --warmup 1 --no-cpu-baseline --no-split --no-check --e2e-steps 1"
for res in device host; do
  timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
     -k regex:"segment|compress|unit_step|score|select|attend" -c 200 --csv --log-file $O/launches_$res.csv \
     python bench.py --residency $res $A > /dev/null 2>&1; echo "launches $res rc=$?"
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:unit_step -s 40 -c 1 \
     -o $O/prof_step_$res python bench.py --residency $res $A > $O/ncu_step_$res.log 2>&1; echo "full $res rc=$?"
done
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"alpha_colsum|alpha_rowstats|retain_topk" -s 3 -c 3 \
   -o $O/prof_retain python scripts/retain_probe.py full > $O/ncu_retain.log 2>&1; echo "retain rc=$?"
ls $O
