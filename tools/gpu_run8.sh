#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_solver.py tests/test_dense_gpu.py tests/test_capi.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest8.txt 2>&1
timeout 900 python bench.py --steps 100 --warmup 10 > gpurun_out/bench8.txt 2>&1
timeout 600 python tools/bench_paths.py multires --n 512 --steps 5 > gpurun_out/paths_mres8.txt 2>&1
tail -3 gpurun_out/pytest8.txt; grep -E "FAIL|Error" gpurun_out/pytest8.txt | head; python -c "
import json; d=json.loads(open('gpurun_out/bench8.txt').read().strip().splitlines()[-1]); print(d['value'], d['e2e'], d['roofline']['frac'])"; cut -c1-260 gpurun_out/paths_mres8.txt
