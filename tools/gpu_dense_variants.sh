#!/bin/bash
# Dense 512^3 step (bench.py value) for each CTA size / bound variant, twice round-robin.
mkdir -p gpurun_out
bash tools/build_dense_variants.sh > gpurun_out/dv_build.txt 2>&1 || { tail gpurun_out/dv_build.txt; exit 1; }
cp paper_2503_07898_b200/_lib/libvoxl_b200.so /tmp/orig.so
for r in 1 2; do
for d in _libvar/d*/; do
  cp $d/libvoxl_b200.so paper_2503_07898_b200/_lib/libvoxl_b200.so
  timeout 300 python bench.py --steps 200 --warmup 20 --no-e2e --no-cpu --no-paths 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d', d['value'], d['roofline']['avg_kernel_ms'], d['clocks']['sm_mhz'])"
done
done
cp /tmp/orig.so paper_2503_07898_b200/_lib/libvoxl_b200.so
