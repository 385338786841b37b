#!/bin/bash
# configs[1] (8b-32k) and configs[3] (8b-256k) bench lines, device residency, N=1.
O=gpurun_out/${TAG:-cfg}; mkdir -p $O
for c in 8b-32k 8b-256k; do
  timeout -s KILL 900 python bench.py --config $c --steps 100 --warmup 10 > $O/bench_$c.txt 2>&1
  python - $O/bench_$c.txt <<'PY'
import json,sys
j=json.loads([x for x in open(sys.argv[1]) if x.startswith('{')][-1])
k=list(j['kernels'].values())[0]
print(j['config']['workload'], 'ms/step', j['ms_per_step'], 'tok/s', j['value'], 'frac', j['roofline']['frac'], 'us/layer', k['avg_us'], 'MB/layer', round(k['bytes_per_launch']/1e6,2), 'e2e', j['e2e']['ms_per_step'], 'split', (j.get('split_calls') or {}).get('ms_per_step'), 'check', (j.get('end_check') or {}).get('ids_bit_exact_and_O_2e-3'), 'cpu', (j.get('cpu_baseline') or {}).get('value'))
PY
done
