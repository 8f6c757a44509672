#!/bin/bash
# Times every libcil.so variant under paper_2203_14742_b200/lib/var on the C2 step's re-check (bench)
# and the C3 max-family re-check (tools/rk_split.py), twice, alternating
L=paper_2203_14742_b200/lib
cp $L/libcil.so /tmp/libcil_product.so
for pass in 1 2; do
  for f in $L/var/libcil_*.so; do
    cp $f $L/libcil.so; touch $L/libcil.so
    python bench.py --steps 200 --no-cpu --no-e2e --no-c4 --no-c6 --no-c7 --no-c3 --no-c5 > /tmp/vb.json 2>/dev/null
    echo "$(basename $f .so) $(python tools/bsum.py /tmp/vb.json | head -1 | cut -c1-150) | $(python tools/rk_split.py 2>&1 | grep maxfam)"
  done
done
cp /tmp/libcil_product.so $L/libcil.so
