# pack/Gram pipeline sweep on C2 (diagnostic): batches x Gram SM budget
for cfg in "1 0" "2 120" "3 120" "4 112" "4 120" "5 120" "5 128" "3 128"; do
  set -- $cfg
  CIL_TC_BATCHES=$1 CIL_TC_GRAM_SMS=$2 timeout 300 python bench.py --steps 100 --warmup 3 --no-e2e --no-cpu --no-c4 > gpurun_out/ov_$1_$2.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ov_$1_$2.json')); print('batches=$1 sms=$2', d['ms_per_step'], 'ms', round(d['value']/1e9,2), 'Gpairs/s', {k:v['ms_per_step'] for k,v in d['kernel_breakdown'].items()})"
done
