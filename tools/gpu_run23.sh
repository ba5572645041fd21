#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/time_probe.py 512 50 > gpurun_out/probe23.txt 2>&1
timeout 300 python tools/time_probe.py 512 50 >> gpurun_out/probe23.txt 2>&1
timeout 900 python -m pytest tests/test_dense_gpu.py tests/test_multires.py tests/test_solver.py tests/test_multigpu.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest23.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_step -s 3 -c 2 -o gpurun_out/probe_full23 python tools/prof_probe.py 512 > /dev/null 2>&1
tail -2 gpurun_out/pytest23.txt; grep -E "^FAILED|^E " gpurun_out/pytest23.txt | head; cat gpurun_out/probe23.txt
