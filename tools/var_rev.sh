#!/bin/bash
# Builds libcil.so variants from two revisions of one source file (the committed one and the working
# tree) into paper_2203_14742_b200/lib/var/ for A/B timing (tools/var_bench.sh):
#   FILE=gram3 [REV=HEAD] bash tools/var_rev.sh
set -e
cd "$(dirname "$0")/.."
L=paper_2203_14742_b200/lib; rm -rf $L/var; mkdir -p $L/var
FILE=${FILE:-gram3}; REV=${REV:-HEAD}
python paper_2203_14742_b200/build.py > /dev/null
others=$(ls $L/obj/*.o | grep -v "/$FILE.cu.o")
git show $REV:paper_2203_14742_b200/csrc/$FILE.cu > paper_2203_14742_b200/csrc/.rev_$FILE.cu
one() {  # tag src
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
    --expt-relaxed-constexpr -Ipaper_2203_14742_b200/csrc -c $2 -o /tmp/var_$1.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $L/var/libcil_$1.so $others /tmp/var_$1.o -Xcompiler -fvisibility=hidden
}
one a_rev paper_2203_14742_b200/csrc/.rev_$FILE.cu & one b_work paper_2203_14742_b200/csrc/$FILE.cu & wait
rm -f paper_2203_14742_b200/csrc/.rev_$FILE.cu
ls $L/var
