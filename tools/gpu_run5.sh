#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_multires.py -q -s -m gpu -p no:cacheprovider > gpurun_out/pytest_mres.txt 2>&1
timeout 600 python tools/bench_paths.py multires --n 256 --steps 10 > gpurun_out/bench_mres256.txt 2>&1
timeout 900 python tools/bench_paths.py multires --n 512 --steps 5 > gpurun_out/bench_mres512.txt 2>&1
tail -15 gpurun_out/pytest_mres.txt; cat gpurun_out/bench_mres256.txt gpurun_out/bench_mres512.txt | cut -c1-600
