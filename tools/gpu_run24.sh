#!/bin/bash
mkdir -p gpurun_out
cp paper_2503_07898_b200/_lib/libvoxl_b200.so /tmp/keep.so
for i in 1 2; do for d in _libvar/*/; do
  tag=$(basename $d)
  cp $d/libvoxl_b200.so paper_2503_07898_b200/_lib/libvoxl_b200.so
  TAG=$tag timeout 300 python tools/time_probe.py 512 100 >> gpurun_out/variants24.txt 2>&1
done; done
cp /tmp/keep.so paper_2503_07898_b200/_lib/libvoxl_b200.so
timeout 600 python tools/e2e_breakdown.py 512 200 > gpurun_out/e2e24.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 3 -c 30 --csv --log-file gpurun_out/launches24.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
cat gpurun_out/variants24.txt gpurun_out/e2e24.txt
