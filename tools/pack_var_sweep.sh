for v in 0 1 2 3; do for pf in 4 8; do echo "VAR=$v PF=$pf"; CIL_PACK_VAR=$v CIL_PACK_PF=$pf timeout 120 python tools/prof_c4.py 2>&1 | tail -1; done; done
