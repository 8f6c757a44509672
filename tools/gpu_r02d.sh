set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_neardup.py -q -x -p no:cacheprovider > gpurun_out/r02d_tests.log 2>&1; tail -3 gpurun_out/r02d_tests.log
python bench.py --no-cpu --no-e2e > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-c4 --no-c6 --no-c7"
$CMD > gpurun_out/r02d_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gram3 -s 3 -c 1 -o gpurun_out/r02d_gram $CMD > gpurun_out/r02d_ncu_gram.log 2>&1; \
ncu --set full --clock-control none --import-source on -k "regex:k_pack3" -s 6 -c 2 -o gpurun_out/r02d_pack $CMD > gpurun_out/r02d_ncu_pack.log 2>&1; echo ncu_rc=$?
