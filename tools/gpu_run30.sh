#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_sparse.py tests/test_multires.py tests/test_fullsize.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest30.txt 2>&1
timeout 600 python tools/bench_paths.py multires --n 512 --steps 5 > gpurun_out/paths_mres30.txt 2>&1
tail -2 gpurun_out/pytest30.txt; grep -E "^FAILED|^E " gpurun_out/pytest30.txt | head; cut -c1-500 gpurun_out/paths_mres30.txt
