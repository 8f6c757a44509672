CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-c4 --no-c6 --no-c7 --no-c3 --no-c5"
$CMD > gpurun_out/r02r_plain.log 2>&1 || { echo plain_failed; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:k_gram3 -s 3 -c 1 -o gpurun_out/r02r_gram $CMD > gpurun_out/r02r_ncu_gram.log 2>&1; echo gram=$?
ncu --set full --clock-control none --import-source on -k "regex:k_pack3|k_center" -s 9 -c 3 -o gpurun_out/r02r_pack $CMD > gpurun_out/r02r_ncu_pack.log 2>&1; echo pack=$?
