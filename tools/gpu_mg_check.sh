#!/bin/bash
# Multi-process dense paths on one B200 (ranks share the GPU): halo modes, stall guard, bench under torchrun.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_multigpu.py tests/test_dense_gpu.py tests/test_capi.py -q -m gpu -p no:cacheprovider > gpurun_out/mg_pytest.txt 2>&1
tail -2 gpurun_out/mg_pytest.txt; grep -E "^FAILED|^E " gpurun_out/mg_pytest.txt | head -20
for h in zero_copy copy; do
VOXL_SHARE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --size 256 --no-cpu --halo $h > gpurun_out/mg_bench_$h.txt 2>&1
tail -1 gpurun_out/mg_bench_$h.txt | cut -c1-400
done
timeout 600 python tools/emulate_rank.py > gpurun_out/emulate.txt 2>&1; tail -5 gpurun_out/emulate.txt
