#!/bin/bash
# Times every libcil.so variant under paper_2203_14742_b200/lib/var: re-check at the C3 and C5 shapes
L=paper_2203_14742_b200/lib
cp $L/libcil.so /tmp/libcil_product.so
for f in $L/var/libcil_*.so; do
  cp $f $L/libcil.so; touch $L/libcil.so
  echo "$(basename $f .so) C3 $(python tools/rk_split.py 2>&1 | grep -E 'L2fam|maxfam' | sed 's/{.*recheck.: \([0-9.]*\).*/recheck \1/' | paste -sd' ')"
  echo "$(basename $f .so) C5 $(python tools/rk_split_c5.py 2>&1 | grep -E 'L2fam|maxfam' | sed 's/{.*recheck.: \([0-9.]*\).*/recheck \1/' | paste -sd' ')"
done
cp /tmp/libcil_product.so $L/libcil.so
