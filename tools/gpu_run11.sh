#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multigpu.py tests/test_dense_gpu.py tests/test_solver.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest11.txt 2>&1
tail -3 gpurun_out/pytest11.txt; grep -E "^FAILED|^ERROR" gpurun_out/pytest11.txt | head
