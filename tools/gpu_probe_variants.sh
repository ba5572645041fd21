#!/bin/bash
# Fused-probe step variants (partials layout, CTA-per-SM bound) timed on one B200: D3Q19 keeps 6 CTAs/SM (3.33 ms vs 3.39 at 5, 3.55-3.60 at 4).
mkdir -p gpurun_out
bash tools/build_variants.sh > gpurun_out/variants_build.txt 2>&1
cp paper_2503_07898_b200/_lib/libvoxl_b200.so /tmp/libvoxl_b200.so.orig
for t in w1 m5 m4 w1 m5 m4; do
  cp _libvar/$t/libvoxl_b200.so paper_2503_07898_b200/_lib/libvoxl_b200.so
  TAG=$t timeout 300 python tools/time_probe.py 512 100 >> gpurun_out/probe_variants.txt 2>&1
done
cp /tmp/libvoxl_b200.so.orig paper_2503_07898_b200/_lib/libvoxl_b200.so
cat gpurun_out/probe_variants.txt
