#!/bin/bash
# A/B build of one translation unit with extra -D flags, linked against the
# regular objects:  tools/build_variant.sh NAME FILE.cu -DFOO=1 ...  ->  build_ab/libedfa_NAME.so
# (run with EDFA_LIB=build_ab/libedfa_NAME.so; build_ab/ is git-ignored but travels to the GPU box)
set -e
name=$1; src=$2; shift 2
cd "$(dirname "$0")/../paper_2009_13916_b200/csrc"
make -s >/dev/null
mkdir -p ../../build_ab
stem=${src%.cu}
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 \
  --expt-relaxed-constexpr -diag-suppress 177 "$@" -c $src -o ../../build_ab/${stem}_$name.o
objs=$(ls build/*.o | grep -v "build/$stem.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared $objs ../../build_ab/${stem}_$name.o -o ../../build_ab/libedfa_$name.so
rm ../../build_ab/${stem}_$name.o
echo build_ab/libedfa_$name.so
