#!/bin/bash
# Gram bottleneck experiment: rebuild libcil.so with CIL_G3_EXP = 0..3 on the GPU box (scratch copy)
# and time the C2 step for each.  tag = $1
tag=${1:-g3exp}
for e in 0 1 2 3; do
  CIL_BUILD_DEFINES="-DCIL_G3_EXP=$e" python paper_2203_14742_b200/build.py --force > /dev/null || exit 1
  python bench.py --steps 50 --no-cpu --no-e2e --no-c4 --no-c6 --no-c7 > gpurun_out/${tag}_$e.json 2>/dev/null
  python tools/bsum.py gpurun_out/${tag}_$e.json | head -1 | sed "s/^/exp=$e /"
done
