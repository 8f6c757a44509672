CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-c4"
$CMD > gpurun_out/plain_i8c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gram_i8 -s 3 -c 1 -o gpurun_out/prof_gram_i8c $CMD > gpurun_out/ncu_full_i8c.log 2>&1
echo full_rc=$?
