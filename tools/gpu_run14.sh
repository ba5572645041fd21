#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multires.py tests/test_sparse.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest14.txt 2>&1
timeout 600 python tools/bench_paths.py multires --n 512 --steps 5 > gpurun_out/paths_mres14.txt 2>&1
timeout 600 python tools/bench_paths.py sparse --n 512 --steps 20 > gpurun_out/paths_sparse14.txt 2>&1
tail -2 gpurun_out/pytest14.txt; grep -E "^FAILED" gpurun_out/pytest14.txt | head; python -c "
import json
for f in ['gpurun_out/paths_mres14.txt','gpurun_out/paths_sparse14.txt']:
  for l in open(f):
    d=json.loads(l); print(d.get('fused', d.get('strategy')), d['MLUPS'], d['frac_of_measured_peak'], d['frac_of_8TBs'])"
