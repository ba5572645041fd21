#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_sparse.py tests/test_multires.py tests/test_fullsize.py tests/test_solver.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest29.txt 2>&1
timeout 600 python tools/time_probe.py 512 100 > gpurun_out/probe29.txt 2>&1
timeout 600 python tools/bench_paths.py sparse --n 512 --steps 20 > gpurun_out/paths_sparse29.txt 2>&1
tail -2 gpurun_out/pytest29.txt; grep -E "^FAILED|^E " gpurun_out/pytest29.txt | head; cat gpurun_out/probe29.txt; cut -c1-250 gpurun_out/paths_sparse29.txt
