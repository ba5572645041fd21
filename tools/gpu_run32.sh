#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_sparse.py tests/test_multires.py tests/test_solver.py tests/test_capi.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest32.txt 2>&1
timeout 900 python tools/run_paths.py > gpurun_out/runpaths32.txt 2>&1
tail -2 gpurun_out/pytest32.txt; grep -E "^FAILED|^E " gpurun_out/pytest32.txt | head -20; cat gpurun_out/runpaths32.txt
