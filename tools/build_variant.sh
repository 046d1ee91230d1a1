#!/bin/bash
# build_ab/libedfa_NAME.so = libedfa.so with FILE.cu recompiled under extra -D flags
# usage: tools/build_variant.sh NAME FILE "-DKNOB=V ..."
set -e
name=$1; file=$2; flags=$3
C=paper_2009_13916_b200/csrc
make -s -C $C >/dev/null
mkdir -p build_ab/$name
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -diag-suppress 177"
$NV $flags -Xptxas -v -c $C/$file.cu -o build_ab/$name/$file.o 2> build_ab/$name/ptxas.txt
objs=$(ls $C/build/*.o | grep -v "/$file.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared $objs build_ab/$name/$file.o -o build_ab/libedfa_$name.so
echo "built build_ab/libedfa_$name.so"
