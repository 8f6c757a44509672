#!/bin/bash
# Builds libcil.so variants that differ only in one source file (code-generation experiments for the
# CUDA-core engines) into paper_2203_14742_b200/lib/var/; tools/simt_var.sh times each on the GPU.
#   FILE=max16 MACRO=CIL_M16_EXP VARIANTS="0 1 2 3" bash tools/simt_var_build.sh
set -e
cd "$(dirname "$0")/.."
L=paper_2203_14742_b200/lib; rm -rf $L/var; mkdir -p $L/var
FILE=${FILE:-simt_tile}; MACRO=${MACRO:-CIL_SIMT_EXP}
python paper_2203_14742_b200/build.py > /dev/null
others=$(ls $L/obj/*.o | grep -v "/$FILE.cu.o")
one() {  # tag src defines...
  tag=$1; src=$2; shift 2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
    --expt-relaxed-constexpr -Ipaper_2203_14742_b200/csrc "$@" -c $src -o /tmp/var_$tag.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $L/var/libcil_$tag.so $others /tmp/var_$tag.o -Xcompiler -fvisibility=hidden
}
for v in ${VARIANTS:-0 1 2 3 4}; do one v$v paper_2203_14742_b200/csrc/$FILE.cu -D$MACRO=$v & done
wait
ls $L/var
