#!/bin/bash
# libvoxl_b200.so variants of the dense step kernel's CTA size / CTA-per-SM bound into _libvar/d<B>_<M>/
set -e
cd "$(dirname "$0")/.."
P=paper_2503_07898_b200
python -c "import __graft_entry__ as g; g._load_builder().build()"
V="${DENSE_VARIANTS:-256:0 512:0 512:3 1024:0 256:5}"
for v in $V; do
  b=${v%%:*}; m=${v##*:}; d=_libvar/d${b}_$m; mkdir -p $d
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-ffp-contract=off,-O3 -Iinclude -DVOXL_DENSE_BLOCK=$b -DVOXL_DENSE_MINB=$m $EXTRA_FLAGS -x cu -c $P/csrc/dense.cu -o $d/dense.o &
done
wait
for v in $V; do
  b=${v%%:*}; m=${v##*:}; d=_libvar/d${b}_$m
  objs=$(ls $P/_lib/obj/*.o | grep -v dense.cu.o)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/libvoxl_b200.so $objs $d/dense.o -lcudart -lcuda
done
ls _libvar/*/libvoxl_b200.so
