#!/bin/bash
# Build libvoxl_b200.so variants of the fused-probe step (partials layout, CTA-per-SM bound) into _libvar/<tag>/
# (tools/time_probe.py times each after it is copied over the in-tree library).
set -e
cd "$(dirname "$0")/.."
P=paper_2503_07898_b200
python -c "import __graft_entry__ as g; g._load_builder().build()"
for v in "w1:-DVOXL_DIAG_WARP=1" "w0:-DVOXL_DIAG_WARP=0" "m5:-DVOXL_DIAG_MINB=5" "m4:-DVOXL_DIAG_MINB=4"; do
  tag=${v%%:*}; defs=${v#*:}
  mkdir -p _libvar/$tag
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-ffp-contract=off,-O3 -Iinclude $defs -x cu -c $P/csrc/dense.cu -o _libvar/$tag/dense.o &
done
wait
for d in _libvar/*/; do
  objs=$(ls $P/_lib/obj/*.o | grep -v dense.cu.o)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/libvoxl_b200.so $objs $d/dense.o -lcudart -lcuda
done
ls _libvar/*/libvoxl_b200.so
