#!/bin/bash
# A/B of the libcil.so variants under paper_2203_14742_b200/lib/var on the C3 line (bench.py --config C3), twice
L=paper_2203_14742_b200/lib
cp $L/libcil.so /tmp/libcil_product.so
for pass in 1 2; do for f in $L/var/libcil_*.so; do cp $f $L/libcil.so; touch $L/libcil.so
  echo "$(basename $f .so) $(python bench.py --config C3 --steps 20 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], d["kernel_breakdown"])')"
done; done
cp /tmp/libcil_product.so $L/libcil.so
