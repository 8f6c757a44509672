for pf in 2 4 6 8 12; do echo "PF=$pf"; CIL_PACK_PF=$pf QB_FLAGS="--no-c6" tools/quick_bench.sh 0; done
