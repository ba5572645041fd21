#!/bin/bash
# Round-2 validation: full GPU suite (no -x), smoke, default bench line, reference arm,
# self-launched 2-rank bench on one GPU, ncu launch list of the bench. Tag = $1.
T=${1:-r2}
mkdir -p gpurun_out
(nproc; nvidia-smi; nvidia-smi topo -m) > gpurun_out/host_$T.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/suite_$T.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_$T.txt 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$T.txt 2>&1
VOXL_SHARE_DEVICE=1 timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench2_$T.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 3 -c 30 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-paths > /dev/null 2>&1
tail -25 gpurun_out/suite_$T.txt; tail -2 gpurun_out/smoke_$T.txt; tail -c 1500 gpurun_out/bench_$T.txt; tail -c 600 gpurun_out/bench_ref_$T.txt; tail -c 800 gpurun_out/bench2_$T.txt
