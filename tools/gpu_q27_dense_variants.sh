#!/bin/bash
mkdir -p gpurun_out
bash tools/build_q27_dense_variants.sh > gpurun_out/qd_build.txt 2>&1 || { tail gpurun_out/qd_build.txt; exit 1; }
cp paper_2503_07898_b200/_lib/libvoxl_b200.so /tmp/orig.so
for r in 1 2; do for d in _libvar/dq*/; do
  cp $d/libvoxl_b200.so paper_2503_07898_b200/_lib/libvoxl_b200.so
  TAG=$d timeout 300 python tools/time_q27_dense.py 2>&1 | tail -1
done; done
cp /tmp/orig.so paper_2503_07898_b200/_lib/libvoxl_b200.so
