#!/bin/bash
# Multires parity suite + the 512^3 multires path bench (D3Q19 and D3Q27).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_multires.py tests/test_solver.py tests/test_fullsize.py -q -m gpu -p no:cacheprovider > gpurun_out/mq_pytest.txt 2>&1
tail -2 gpurun_out/mq_pytest.txt; grep -E "^FAILED|^E " gpurun_out/mq_pytest.txt | head -20
timeout 600 python tools/bench_paths.py multires --n 512 --steps 5 > gpurun_out/mq_paths.txt 2>&1
timeout 600 python tools/bench_paths.py multires --n 512 --steps 3 --lattice D3Q27 > gpurun_out/mq_paths27.txt 2>&1
cut -c1-420 gpurun_out/mq_paths.txt gpurun_out/mq_paths27.txt
