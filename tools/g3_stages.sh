#!/bin/bash
# A/B of the INT8 Gram pipeline depth: 3 vs 2 stages (build-time CIL_G3_MAXSTAGES)
tag=${1:-g3st}
for d in "" "-DCIL_G3_MAXSTAGES=2"; do
  CIL_BUILD_DEFINES="$d" python paper_2203_14742_b200/build.py --force > /dev/null || exit 1
  python bench.py --steps 100 --no-cpu --no-e2e --no-c6 --no-c7 --no-c5 > gpurun_out/${tag}.json 2>/dev/null
  python tools/bsum.py gpurun_out/${tag}.json | head -1 | sed "s/^/[$d] /"
  python tools/bsum.py gpurun_out/${tag}.json | grep secondary | sed "s/^/[$d] /"
done
