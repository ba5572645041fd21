#!/bin/bash
# first B200 session: environment facts, smoke, GPU parity tests, bench, ncu
mkdir -p gpurun_out
{
nvidia-smi; free -g; nproc; lscpu | grep -E "Model name|Socket|Thread|Core"
} > gpurun_out/env.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
timeout 600 python bench.py --steps 100 --warmup 10 --no-e2e > gpurun_out/bench1.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu > gpurun_out/ncu_launch_stdout.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_step -s 2 -c 1 -o gpurun_out/dense_full python tools/prof_dense.py 512 4 > gpurun_out/ncu_full_stdout.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt; cat gpurun_out/bench1.txt | tail -2
