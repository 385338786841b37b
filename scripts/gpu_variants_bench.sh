#!/bin/bash
# Bench lines of the NEXT rows at 8b-128k, device residency (one line each), for profiles/.
O=gpurun_out/${TAG:-vb}; mkdir -p $O
A="--residency device --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 10"
for v in "--retention" "--buckets equal" "--outlier-n 1.0" "--query current" "--fill skip" "--buckets quest --page 16" "--buckets quest --page 32"; do
  n=$(echo $v | tr -d ' -')
  timeout -s KILL 600 python bench.py $A $v > $O/bench_$n.txt 2>&1
  python - $O/bench_$n.txt <<'PY'
import json,sys
try:
    j=json.loads([x for x in open(sys.argv[1]) if x.startswith('{')][-1])
    k=list(j['kernels'].values())[0]
    print(j['config']['workload'], 'ms/step', j['ms_per_step'], 'tok/s', j['value'], 'frac', j['roofline']['frac'], 'us/layer', k['avg_us'], 'MB/layer', round(k['bytes_per_launch']/1e6,2), 'launches/step', j['gpu_launches']//j['steps'], 'split', (j.get('split_calls') or {}).get('ms_per_step'), 'ret', j.get('retention'))
except Exception as e: print(sys.argv[1], 'FAILED', e, open(sys.argv[1]).read()[-1500:])
PY
done
