#!/bin/bash
# Dense fast-path cache hints: plain vs st.global.cs stores vs ld.global.lu loads (512^3 bench value, 3 rounds).
mkdir -p gpurun_out
cd "$(dirname "$0")/.."
P=paper_2503_07898_b200
python -c "import __graft_entry__ as g; g._load_builder().build()"
for v in "base:" "stcs:-DVOXL_ST_HINT=1" "ldlu:-DVOXL_LD_HINT=1" "both:-DVOXL_ST_HINT=1 -DVOXL_LD_HINT=1"; do
  t=${v%%:*}; f=${v#*:}; d=_libvar/h_$t; mkdir -p $d
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-ffp-contract=off,-O3 -Iinclude $f -x cu -c $P/csrc/dense.cu -o $d/dense.o &
done
wait
for d in _libvar/h_*; do
  objs=$(ls $P/_lib/obj/*.o | grep -v dense.cu.o)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/libvoxl_b200.so $objs $d/dense.o -lcudart -lcuda
done
cp $P/_lib/libvoxl_b200.so /tmp/orig.so
for r in 1 2 3; do for d in _libvar/h_*; do
  cp $d/libvoxl_b200.so $P/_lib/libvoxl_b200.so
  timeout 300 python bench.py --steps 200 --warmup 20 --no-e2e --no-cpu --no-paths 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d', d['value'], d['roofline']['avg_kernel_ms'], d['clocks']['sm_mhz'])"
done; done
cp /tmp/orig.so $P/_lib/libvoxl_b200.so
