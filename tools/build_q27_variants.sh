#!/bin/bash
# libvoxl_b200.so variants of the D3Q27 8^3-block kernels' CTA-per-SM bound into _libvar/q27m<N>/
set -e
cd "$(dirname "$0")/.."
P=paper_2503_07898_b200
python -c "import __graft_entry__ as g; g._load_builder().build()"
for m in 6 5 4; do
  mkdir -p _libvar/q27m$m
  for src in sparse multires; do
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-ffp-contract=off,-O3 -Iinclude -DVOXL_BLOCK_MINB27=$m -x cu -c $P/csrc/$src.cu -o _libvar/q27m$m/$src.o &
  done
done
wait
for m in 6 5 4; do
  objs=$(ls $P/_lib/obj/*.o | grep -v -e sparse.cu.o -e multires.cu.o)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o _libvar/q27m$m/libvoxl_b200.so $objs _libvar/q27m$m/sparse.o _libvar/q27m$m/multires.o -lcudart -lcuda
done
ls _libvar/q27m*/libvoxl_b200.so
