#!/bin/bash
for pf in 0 2 4 8; do echo "I8_PF=$pf"; CIL_I8_PF=$pf QB_FLAGS="--no-c6" tools/quick_bench.sh 0; done
