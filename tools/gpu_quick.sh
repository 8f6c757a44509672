#!/bin/bash
# quick GPU check: core parity tests + the bench (C2 headline + secondaries); tag = $1
tag=${1:-q}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_neardup.py -q -x -p no:cacheprovider > gpurun_out/${tag}_tests.log 2>&1; tail -2 gpurun_out/${tag}_tests.log
python bench.py --no-cpu --no-e2e > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo bench_rc=$?
