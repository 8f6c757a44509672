#!/bin/bash
# Times every libcil.so variant under paper_2203_14742_b200/lib/var (tools/simt_var_build.sh) on the C2
# step and the C4 line, twice, alternating (bench.py, summarised by tools/bsum.py)
L=paper_2203_14742_b200/lib
cp $L/libcil.so /tmp/libcil_product.so
for pass in 1 2; do
  for f in $L/var/libcil_*.so; do
    cp $f $L/libcil.so; touch $L/libcil.so
    python bench.py --steps 200 --no-cpu --no-e2e --no-c6 --no-c7 --no-c3 --no-c5 > /tmp/vb.json 2>/dev/null
    python tools/bsum.py /tmp/vb.json | grep -v roofline | sed "s/^/$(basename $f .so) /" | cut -c1-200
  done
done
cp /tmp/libcil_product.so $L/libcil.so
