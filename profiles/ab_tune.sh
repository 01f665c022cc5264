for t in "zero_async=8" "zero_async=0" "zero_async=2" "zero_async=16"; do
  SVR_TUNING=$t timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extra > gpurun_out/t.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/t.json')); r=d['roofline']
print('$t', 'ms/step %.3f'%d['ms_per_step'], 'fwd_call %.3f'%r['fwd_call_ms'], 'bwd %.3f'%r['bwd_ms'])"
done
