#!/bin/bash
mkdir -p gpurun_out
nproc > gpurun_out/host20.txt; lscpu | grep -E "Model name|Socket|Core|Thread|NUMA node" >> gpurun_out/host20.txt; free -g >> gpurun_out/host20.txt
timeout 600 python -m pytest tests/test_dense_gpu.py tests/test_fullsize.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest20.txt 2>&1
timeout 600 python tools/e2e_breakdown.py 512 200 > gpurun_out/e2e20.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/probe20.csv python tools/prof_probe.py 512 > /dev/null 2>&1
tail -2 gpurun_out/pytest20.txt; cat gpurun_out/e2e20.txt gpurun_out/host20.txt; grep -v "^==" gpurun_out/probe20.csv | cut -d, -f5,15,16 | tail -30
