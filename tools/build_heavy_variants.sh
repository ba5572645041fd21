#!/bin/bash
# libvoxl_b200.so variants of the block-sparse heavy kernel's CTA-per-SM bound into _libvar/h<N>/
set -e
cd "$(dirname "$0")/.."
P=paper_2503_07898_b200
python -c "import __graft_entry__ as g; g._load_builder().build()"
for m in 1 4; do
  mkdir -p _libvar/h$m
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-ffp-contract=off,-O3 -Iinclude -DVOXL_HEAVY_MINB=$m -x cu -c $P/csrc/sparse.cu -o _libvar/h$m/sparse.o &
done
wait
for m in 1 4; do
  objs=$(ls $P/_lib/obj/*.o | grep -v -e sparse.cu.o)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o _libvar/h$m/libvoxl_b200.so $objs _libvar/h$m/sparse.o -lcudart -lcuda
done
