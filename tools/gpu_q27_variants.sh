#!/bin/bash
# D3Q27 block-sparse and multires paths at 512^3 for each CTA-per-SM bound (and D3Q19 as the control).
mkdir -p gpurun_out
bash tools/build_q27_variants.sh > gpurun_out/q27_build.txt 2>&1
cp paper_2503_07898_b200/_lib/libvoxl_b200.so /tmp/libvoxl_b200.so.orig
for m in 6 5 4; do
  cp _libvar/q27m$m/libvoxl_b200.so paper_2503_07898_b200/_lib/libvoxl_b200.so
  echo "== q27 minb $m" >> gpurun_out/q27_paths.txt
  timeout 600 python tools/bench_paths.py sparse --n 512 --steps 10 --lattice D3Q27 >> gpurun_out/q27_paths.txt 2>&1
  timeout 600 python tools/bench_paths.py multires --n 512 --steps 3 --lattice D3Q27 >> gpurun_out/q27_paths.txt 2>&1
done
cp /tmp/libvoxl_b200.so.orig paper_2503_07898_b200/_lib/libvoxl_b200.so
python - <<'PY'
import json
for l in open("gpurun_out/q27_paths.txt"):
    if l.startswith("=="): print(l.strip()); continue
    if not l.startswith("{"): continue
    d = json.loads(l)
    print(d["path"], d.get("strategy", d.get("scenario")), d.get("fused", ""), d["MLUPS"], d["frac_of_measured_peak"])
PY
