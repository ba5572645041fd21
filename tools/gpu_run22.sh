#!/bin/bash
mkdir -p gpurun_out
cp paper_2503_07898_b200/_lib/libvoxl_b200.so /tmp/keep.so
for d in _libvar/*/; do
  tag=$(basename $d)
  cp $d/libvoxl_b200.so paper_2503_07898_b200/_lib/libvoxl_b200.so
  TAG=$tag timeout 300 python tools/time_probe.py 512 50 >> gpurun_out/variants22.txt 2>&1
  TAG=$tag timeout 300 python tools/time_probe.py 512 50 >> gpurun_out/variants22.txt 2>&1
done
cp /tmp/keep.so paper_2503_07898_b200/_lib/libvoxl_b200.so
timeout 900 python -m pytest tests/test_dense_gpu.py tests/test_multires.py tests/test_solver.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest22.txt 2>&1
tail -2 gpurun_out/pytest22.txt; cat gpurun_out/variants22.txt
