#!/bin/bash
# quick C2 / C4 / C6 kernel breakdown: CIL_DEBUG_I8 = 0 (full), 1 (no binning), ...; args: debug levels
for d in "${@:-0}"; do
  CIL_DEBUG_I8=$d timeout 300 python bench.py --steps 100 --warmup 3 --no-e2e --no-cpu $QB_FLAGS 2>/dev/null | tail -1 | python -c "
import json,sys; j=json.loads(sys.stdin.read())
print('dbg=$d', round(j['value']/1e9,3), 'Gpairs/s', j['ms_per_step'], 'ms', {k:v['ms_per_step'] for k,v in j.get('kernel_breakdown',{}).items()})
for key in ('secondary', 'secondary_bootstrap', 'secondary_train'):
    s=j.get(key)
    if isinstance(s, dict): print('  ', s['workload'][:3], s.get('value'), s.get('ms_per_step'), s.get('kernel_breakdown'), s.get('gram_tc', {}).get('frac_of_peak'), s.get('resample'))"
done
