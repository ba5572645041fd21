#!/bin/bash
# libvoxl_b200.so with one translation unit rebuilt under extra -D flags:
#   build_lib_variant.sh NAME SOURCE "-DFOO=1 -DBAR=2"  ->  _libvar/NAME/libvoxl_b200.so
set -e
cd "$(dirname "$0")/.."
P=paper_2503_07898_b200
N=$1; SRC=$2; FL=$3
d=_libvar/$N; mkdir -p $d
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC,-ffp-contract=off,-O3 -Iinclude $FL -x cu -c $P/csrc/$SRC -o $d/${SRC}.o -Xptxas -v 2> $d/ptxas.txt
objs=$(ls $P/_lib/obj/*.o | grep -v "/${SRC}.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/libvoxl_b200.so $objs $d/${SRC}.o -lcudart -lcuda -ldl
echo $d/libvoxl_b200.so
