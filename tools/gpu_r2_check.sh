#!/bin/bash
# Round-2 validation: full GPU suite, smoke, default bench line, self-launched 2-rank bench on one GPU.
mkdir -p gpurun_out
(nproc; nvidia-smi; nvidia-smi topo -m) > gpurun_out/r2_host.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_suite.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/r2_bench.txt 2>&1
VOXL_SHARE_DEVICE=1 timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_bench2.txt 2>&1
tail -3 gpurun_out/r2_suite.txt; tail -2 gpurun_out/r2_smoke.txt; tail -c 1500 gpurun_out/r2_bench.txt; tail -c 800 gpurun_out/r2_bench2.txt
