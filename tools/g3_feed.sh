#!/bin/bash
# Gram operand-feed experiment: rebuild libcil.so with CIL_G3_EXP = 0 (product), 4 (B loads only),
# 8 (A loads only), 1 (no epilogue drain) and time the C2 step and the C4 line for each (counts are
# garbage in the experiment builds; timing only).  tag = $1
tag=${1:-g3feed}
for e in 0 4 8 1 0; do
  CIL_BUILD_DEFINES="-DCIL_G3_EXP=$e" python paper_2203_14742_b200/build.py --force > /dev/null || exit 1
  python bench.py --steps 100 --no-cpu --no-e2e --no-c6 --no-c7 --no-c3 --no-c5 > gpurun_out/${tag}_$e.json 2>/dev/null
  python tools/bsum.py gpurun_out/${tag}_$e.json | grep -v roofline | sed "s/^/exp=$e /"
done
