#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dense_gpu.py tests/test_sparse.py tests/test_multires.py tests/test_solver.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest21.txt 2>&1
timeout 600 python tools/e2e_breakdown.py 512 200 > gpurun_out/e2e21.txt 2>&1
timeout 600 python tools/bench_paths.py sparse --n 512 --steps 20 > gpurun_out/paths_sparse21.txt 2>&1
timeout 600 python tools/bench_paths.py multires --n 512 --steps 5 > gpurun_out/paths_mres21.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/probe21.csv python tools/prof_probe.py 512 > /dev/null 2>&1
tail -3 gpurun_out/pytest21.txt; grep -E "^FAILED|rel err" gpurun_out/pytest21.txt | head; cat gpurun_out/e2e21.txt; cut -c1-420 gpurun_out/paths_sparse21.txt gpurun_out/paths_mres21.txt
