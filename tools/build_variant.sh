#!/bin/bash
# build_variant.sh NAME "-DX=.. -DY=.." : a libtk_b200.so variant with extra defines on every source
# (A/B experiments; e.g. "-DTK_DEBUG_KNOBS" makes the library read its TK_* tuning knobs from the
# environment). Load it with TK_LIB_PATH=_variants/libtk_NAME.so.
set -e
cd "$(dirname "$0")/.."
mkdir -p _variants/$1
SRC=paper_2508_10076_b200/csrc
FLAGS="-O3 -std=c++17 -lineinfo -Xcompiler -fPIC -gencode arch=compute_100a,code=sm_100a $2"
objs=""
for f in $(python -c "from paper_2508_10076_b200 import build; print(' '.join(build.SOURCES))"); do
  /usr/local/cuda/bin/nvcc $FLAGS -c $SRC/$f -o _variants/$1/$f.o &
  objs="$objs _variants/$1/$f.o"
done
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o _variants/libtk_$1.so $objs -cudart static
echo _variants/libtk_$1.so
