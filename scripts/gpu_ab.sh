#!/bin/bash
# A/B of library variants on the bench (host residency unless RES is set): VARIANTS="a b" -> libsentencekv_{a,b}.so ("base" = product)
TAG=${TAG:-ab}; O=gpurun_out/$TAG; mkdir -p $O
ARGS=${ARGS:-"--steps 100 --warmup 5 --no-cpu-baseline --no-split --no-check --e2e-steps 10"}
for rep in 1 2; do for v in $VARIANTS; do
  if [ "$v" = base ]; then L=paper_2504_00970_b200/libsentencekv.so; else L=paper_2504_00970_b200/libsentencekv_$v.so; fi
  SKV_LIB=$L timeout 600 python bench.py $ARGS > $O/${v}_$rep.txt 2>&1
  python - $O/${v}_$rep.txt $v <<'PY'
import json,sys
try:
    j=json.loads([x for x in open(sys.argv[1]) if x.startswith('{')][-1])
    h=j.get('host_residency') or {}
    print(sys.argv[2], 'ms/step', j['ms_per_step'], 'p50', j['step_ms']['p50'], 'p90', j['step_ms']['p90'], 'frac', j['roofline']['frac'], 'hostMB/step', round(h.get('host_bytes_per_step',0)/1e6,1), 'cold', h.get('cold_first_step'))
except Exception as e: print(sys.argv[2], 'FAILED', e, open(sys.argv[1]).read()[-800:])
PY
done; done
