#!/bin/bash
# ncu source-level capture of the CUDA-core max family (C3 bench configuration)
CMD="python bench.py --config C3 --steps 2"
$CMD > gpurun_out/simt_plain.log 2>&1 || { echo plain_failed; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:k_simt -s 2 -c 1 -o gpurun_out/r02t_simt $CMD > gpurun_out/r02t_ncu.log 2>&1; echo ncu=$?
