CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-c4"
$CMD > gpurun_out/plain_i8.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_i8.csv $CMD > gpurun_out/ncu_launch_i8.log 2>&1
echo launches_rc=$?
$CMD > gpurun_out/plain_i8b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gram_i8 -s 3 -c 1 -o gpurun_out/prof_gram_i8 $CMD > gpurun_out/ncu_full_i8.log 2>&1
echo full_rc=$?
$CMD > gpurun_out/plain_i8c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pack_i8 -s 6 -c 2 -o gpurun_out/prof_pack_i8 $CMD > gpurun_out/ncu_pack_i8.log 2>&1
echo pack_rc=$?
