#!/bin/bash
# A/B of the CUDA-core engine's rigorous epilogue bound (build-time experiment switch): C3 lines,
# alternating builds so clock ramps / thermal drift show up as A-B-A inconsistency
for d in "-DCIL_SIMT_NOBOUND" "" "-DCIL_SIMT_NOBOUND" ""; do
  CIL_BUILD_DEFINES="$d" python paper_2203_14742_b200/build.py --force > /dev/null || exit 1
  python bench.py --config C3 --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$d] C3', d['ms_per_step'], d['kernel_breakdown'].get('simt_tile'), d['simt_tile']['frac'], d['clocks'])"
done
python paper_2203_14742_b200/build.py --force > /dev/null
