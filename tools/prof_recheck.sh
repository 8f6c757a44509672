#!/bin/bash
# ncu source-level capture of the re-check kernel in the C3 bench configuration
python bench.py --config C3 --steps 2 > /dev/null 2>&1 || { echo plain_failed; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:k_recheck -s 2 -c 1 -o gpurun_out/r02t_recheck python bench.py --config C3 --steps 2 > gpurun_out/r02t_ncu_rk.log 2>&1; echo ncu=$?
