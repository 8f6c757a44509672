#!/bin/bash
# One ncu pass per gpurun call (each after the same command exits 0 without ncu):
#   tools/prof_round.sh launches|gram|pack|c3launches|max16|recheck  [tag]
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-c4 --no-c6 --no-c7 --no-c3 --no-c5"
what=$1; tag=${2:-r01}
case $what in c3launches|max16|recheck) CMD="python bench.py --config C3 --steps 2" ;; esac
mkdir -p gpurun_out
$CMD > gpurun_out/${tag}_plain_${what}.log 2>&1 || { echo plain_failed; exit 1; }
case $what in
  launches)
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
        $CMD > gpurun_out/${tag}_ncu_launches.log 2>&1 ;;
  gram)
    ncu --set full --clock-control none --import-source on -k regex:k_gram3 -s 3 -c 1 \
        -o gpurun_out/${tag}_gram $CMD > gpurun_out/${tag}_ncu_gram.log 2>&1 ;;
  pack)
    ncu --set full --clock-control none --import-source on -k "regex:k_pack3|k_center" -s 9 -c 3 \
        -o gpurun_out/${tag}_pack $CMD > gpurun_out/${tag}_ncu_pack.log 2>&1 ;;
  c3launches)
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_c3_launches.csv \
        $CMD > gpurun_out/${tag}_ncu_c3launches.log 2>&1 ;;
  max16)
    ncu --set full --clock-control none --import-source on -k regex:k_max16_reg -s 3 -c 1 \
        -o gpurun_out/${tag}_max16 $CMD > gpurun_out/${tag}_ncu_max16.log 2>&1 ;;
  recheck)
    ncu --set full --clock-control none --import-source on -k regex:k_recheck -s 1 -c 1 \
        -o gpurun_out/${tag}_recheck $CMD > gpurun_out/${tag}_ncu_recheck.log 2>&1 ;;
esac
echo ${what}_rc=$?
