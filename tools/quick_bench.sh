#!/bin/bash
# quick C2/C4 kernel breakdown: CIL_DEBUG_I8 = 0 (full), 1 (no binning); args: list of debug levels
for d in "${@:-0}"; do
  CIL_DEBUG_I8=$d timeout 200 python bench.py --steps 100 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; j=json.loads(sys.stdin.read())
print('dbg=$d', round(j['value']/1e9,3), 'Gpairs/s', j['ms_per_step'], 'ms', {k:v['ms_per_step'] for k,v in j.get('kernel_breakdown',{}).items()})
s=j.get('secondary'); print('  C4', s.get('ms_per_step') if isinstance(s,dict) else s, s.get('kernel_breakdown') if isinstance(s,dict) else '')"
done
