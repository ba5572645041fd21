#!/bin/bash
mkdir -p gpurun_out
bash tools/build_heavy_variants.sh > gpurun_out/hv_build.txt 2>&1
cp paper_2503_07898_b200/_lib/libvoxl_b200.so /tmp/orig.so
for m in 1 4 1 4; do
  cp _libvar/h$m/libvoxl_b200.so paper_2503_07898_b200/_lib/libvoxl_b200.so
  for lat in D3Q19 D3Q27; do
    timeout 600 python tools/bench_paths.py sparse --n 512 --steps 20 --lattice $lat 2>&1 | grep disag_mem | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('h$m', d['lattice'], d['MLUPS'], d['boundary_kernel_ms'], d['light_kernel_ms'])"
  done
done
cp /tmp/orig.so paper_2503_07898_b200/_lib/libvoxl_b200.so
