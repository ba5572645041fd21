#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sparse.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest_sparse4.txt 2>&1
timeout 600 python tools/bench_paths.py sparse --n 512 --steps 20 > gpurun_out/bench_sparse512_4.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:sparse_step -c 6 python tools/bench_paths.py sparse --n 256 --steps 1 --warmup 0 > gpurun_out/ncu_sparse4.txt 2>&1
tail -2 gpurun_out/pytest_sparse4.txt; cut -c1-330 gpurun_out/bench_sparse512_4.txt
