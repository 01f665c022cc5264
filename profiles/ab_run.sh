#!/bin/bash
# Time side-by-side variants on one box: bash profiles/ab_run.sh "A B C" [rounds]
O=gpurun_out; mkdir -p $O
for r in $(seq 1 ${2:-2}); do
  for v in $1; do
    SVR_LIB_VARIANT=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extra ${BENCH_ARGS} > $O/ab_$v.json 2>$O/ab_$v.err || { echo "$v FAILED"; tail -5 $O/ab_$v.err; continue; }
    python -c "
import json; d=json.load(open('$O/ab_$v.json')); r=d['roofline']
print('$v', 'round $r', 'ms/step %.3f'%d['ms_per_step'], 'fwd_call %.3f'%r['fwd_call_ms'], 'bwd %.3f'%r['bwd_ms'], 'parity', d.get('parity',{}).get('green'))"
  done
done
