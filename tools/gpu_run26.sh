#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/e2e_breakdown.py 512 200 > gpurun_out/e2e26.txt 2>&1
timeout 900 python -m pytest tests/test_dense_gpu.py tests/test_solver.py tests/test_capi.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest26.txt 2>&1
timeout 900 python tools/bench_paths.py dense --n 512 --steps 50 > gpurun_out/paths_dense26.txt 2>&1
tail -2 gpurun_out/pytest26.txt; grep -E "^FAILED|^E " gpurun_out/pytest26.txt | head; cat gpurun_out/e2e26.txt gpurun_out/paths_dense26.txt
