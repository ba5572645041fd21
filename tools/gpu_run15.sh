#!/bin/bash
# round-1 re-entry: full GPU suite, smoke, bench (both arms), 2-rank shared-device bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi15.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest15.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke15.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench15.txt 2>&1
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref15.txt 2>&1
VOXL_SHARE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --size 256 --no-e2e --no-cpu > gpurun_out/bench_2r15.txt 2>&1
tail -3 gpurun_out/pytest15.txt; grep -E "^FAILED|Error" gpurun_out/pytest15.txt | head
tail -2 gpurun_out/smoke15.txt; tail -1 gpurun_out/bench15.txt | cut -c1-600; tail -1 gpurun_out/bench_ref15.txt | cut -c1-400; tail -1 gpurun_out/bench_2r15.txt | cut -c1-300
