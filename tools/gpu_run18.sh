#!/bin/bash
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi18.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x --durations=15 > gpurun_out/pytest18.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke18.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench18.txt 2>&1
tail -20 gpurun_out/pytest18.txt; tail -2 gpurun_out/smoke18.txt; tail -1 gpurun_out/bench18.txt
