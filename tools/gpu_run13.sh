#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multires.py tests/test_solver.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest13.txt 2>&1
timeout 600 python tools/bench_paths.py multires --n 512 --steps 5 > gpurun_out/paths_mres13.txt 2>&1
tail -2 gpurun_out/pytest13.txt; grep -E "^FAILED" gpurun_out/pytest13.txt | head; python -c "
import json
for l in open('gpurun_out/paths_mres13.txt'):
    d=json.loads(l); print(d['fused'], d['MLUPS'], d['frac_of_measured_peak'], d['frac_of_8TBs'], d['kernels_ms'])"
