#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_fullsize.py -v -m gpu -p no:cacheprovider --durations=0 > gpurun_out/pytest16.txt 2>&1
timeout 600 python tools/e2e_breakdown.py 512 200 > gpurun_out/e2e16.txt 2>&1
tail -25 gpurun_out/pytest16.txt; cat gpurun_out/e2e16.txt | tail -3
