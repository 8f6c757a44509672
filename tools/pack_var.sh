#!/bin/bash
# Times every libcil.so variant under paper_2203_14742_b200/lib/var with tools/pack_var.py, alternating
L=paper_2203_14742_b200/lib
cp $L/libcil.so /tmp/libcil_product.so
for pass in 1 2; do
  for f in $L/var/libcil_*.so; do
    cp $f $L/libcil.so; touch $L/libcil.so
    python tools/pack_var.py $(basename $f .so) 2>&1 | tail -1
  done
done
cp /tmp/libcil_product.so $L/libcil.so
