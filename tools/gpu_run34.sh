#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_sparse.py tests/test_solver.py tests/test_capi.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest34.txt 2>&1
timeout 900 python tools/run_paths.py > gpurun_out/runpaths34.txt 2>&1
timeout 600 python tools/bench_paths.py sparse --n 512 --steps 20 > gpurun_out/paths_sparse34.txt 2>&1
tail -2 gpurun_out/pytest34.txt; grep -E "^FAILED|^E " gpurun_out/pytest34.txt | head -20; cat gpurun_out/runpaths34.txt; cut -c1-300 gpurun_out/paths_sparse34.txt
