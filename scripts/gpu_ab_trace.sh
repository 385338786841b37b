#!/bin/bash
# A/B of step-kernel variants + per-CTA phase traces (trace build): synthetic steady q, then the
# bench's decode script; with TRACE_ENV set, the script trace again under that environment
mkdir -p gpurun_out
bash scripts/gpu_ab.sh "$@"
timeout 300 python scripts/trace_unit.py > gpurun_out/trace_unit.txt 2>&1; grep "span\|modes\|durations" gpurun_out/trace_unit.txt | tail -6
timeout 300 python scripts/trace_unit.py script > gpurun_out/trace_unit_script.txt 2>&1; grep "span\|modes\|durations" gpurun_out/trace_unit_script.txt | tail -24
if [ -n "$TRACE_ENV" ]; then
  env $TRACE_ENV timeout 300 python scripts/trace_unit.py script > gpurun_out/trace_unit_alt.txt 2>&1; echo "== $TRACE_ENV"; grep "span\|modes" gpurun_out/trace_unit_alt.txt | tail -16
fi
