#!/bin/bash
L=paper_2203_14742_b200/lib
cp $L/libcil.so /tmp/libcil_product.so
for f in $L/var/libcil_*.so; do
  cp $f $L/libcil.so; touch $L/libcil.so
  python tools/simt_c3.py $(basename $f .so) 2>&1 | tail -2
done
cp /tmp/libcil_product.so $L/libcil.so
