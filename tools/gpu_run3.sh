#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build3.txt 2>&1
timeout 900 python -m pytest tests/test_sparse.py -q -s -m gpu -p no:cacheprovider > gpurun_out/pytest_sparse.txt 2>&1
timeout 600 python tools/bench_paths.py sparse --n 256 --steps 50 > gpurun_out/bench_sparse256.txt 2>&1
timeout 600 python tools/bench_paths.py sparse --n 512 --steps 20 > gpurun_out/bench_sparse512.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_registers,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,lts__t_bytes.sum --clock-control none -k regex:sparse_step -c 6 python tools/bench_paths.py sparse --n 256 --steps 1 --warmup 0 > gpurun_out/ncu_sparse.txt 2>&1
tail -5 gpurun_out/pytest_sparse.txt; cat gpurun_out/bench_sparse256.txt gpurun_out/bench_sparse512.txt | cut -c1-400
