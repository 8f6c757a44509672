#!/bin/bash
# Times every libcil.so variant under paper_2203_14742_b200/lib/var on the C3 max-family re-check
L=paper_2203_14742_b200/lib
cp $L/libcil.so /tmp/libcil_product.so
for f in $L/var/libcil_*.so; do
  cp $f $L/libcil.so; touch $L/libcil.so
  echo "$(basename $f .so) $(python tools/rk_split.py 2>&1 | grep maxfam)"
done
cp /tmp/libcil_product.so $L/libcil.so
