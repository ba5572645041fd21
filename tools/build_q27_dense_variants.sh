#!/bin/bash
# libvoxl_b200.so variants of the D3Q27 dense step bounds into _libvar/dq<plain>_<diag>/
set -e
cd "$(dirname "$0")/.."
P=paper_2503_07898_b200
python -c "import __graft_entry__ as g; g._load_builder().build()"
V="0:6 5:6 5:5 4:5"
for v in $V; do
  a=${v%%:*}; b=${v##*:}; d=_libvar/dq${a}_$b; mkdir -p $d
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-ffp-contract=off,-O3 -Iinclude -DVOXL_DENSE_MINB27=$a -DVOXL_DIAG_MINB27=$b -x cu -c $P/csrc/dense.cu -o $d/dense.o &
done
wait
for v in $V; do
  a=${v%%:*}; b=${v##*:}; d=_libvar/dq${a}_$b
  objs=$(ls $P/_lib/obj/*.o | grep -v dense.cu.o)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/libvoxl_b200.so $objs $d/dense.o -lcudart -lcuda
done
