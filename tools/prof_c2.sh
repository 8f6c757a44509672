set -x
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-c4"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo launches_rc=$?
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gram_tc -s 3 -c 1 -o gpurun_out/prof_gram $CMD > gpurun_out/ncu_full.log 2>&1
echo full_rc=$?
$CMD > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pack_tc -s 6 -c 2 -o gpurun_out/prof_pack $CMD > gpurun_out/ncu_pack.log 2>&1
echo pack_rc=$?
