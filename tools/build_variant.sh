#!/bin/bash
# build_variant.sh NAME "-DX=.. -DY=.." : libtk_b200.so variant with extra defines for tk_kernels.cu
# (A/B experiments: run with TK_LIB_PATH=_variants/libtk_NAME.so)
set -e
cd "$(dirname "$0")/.."
python -m paper_2508_10076_b200.build >/dev/null
B=paper_2508_10076_b200/_build; mkdir -p _variants
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -gencode arch=compute_100a,code=sm_100a $2 \
  -Xptxas -v -c paper_2508_10076_b200/csrc/tk_kernels.cu -o _variants/k_$1.o 2> _variants/k_$1.log
objs=$(ls $B/*.o | grep -v tk_kernels.cu.o)
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o _variants/libtk_$1.so $objs _variants/k_$1.o -cudart static
echo _variants/libtk_$1.so
