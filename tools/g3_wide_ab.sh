#!/bin/bash
# A/B of the INT8 Gram's MMA layout (CIL_G3_WIDE 0: six N = TN MMAs; 1: four wide MMAs) on the C2
# headline and the C4 / C6 secondaries; variants from tools/simt_var_build.sh (FILE=gram3)
L=paper_2203_14742_b200/lib
cp $L/libcil.so /tmp/libcil_product.so
for pass in 1 2; do
  for f in $L/var/libcil_*.so; do
    cp $f $L/libcil.so; touch $L/libcil.so
    python bench.py --steps 10 --no-e2e --no-cpu --no-c7 --no-c3 --no-c5 2>/dev/null > /tmp/ab.json
    echo "$(basename $f .so) $(python tools/bsum.py /tmp/ab.json | grep -E '^C2|C4|C6' | cut -c1-160 | paste -sd'|')"
  done
done
cp /tmp/libcil_product.so $L/libcil.so
