#!/bin/bash
# bench.py at N=4 and N=8 ranks sharing one B200 at the full 512^3 size (VOXL_SHARE_DEVICE=1):
# the multi-rank code path end to end at the real buffer sizes (timings are time-sliced, not meaningful).
mkdir -p gpurun_out
for n in 4 8; do for h in zero_copy copy; do
VOXL_SHARE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --steps 10 --warmup 3 --no-cpu --halo $h > gpurun_out/mgf_${n}_$h.txt 2>&1
echo "N=$n $h rc=$?"; tail -1 gpurun_out/mgf_${n}_$h.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['config']['halo'], d['diag'], d['e2e'].get('final_mass'), d['e2e'].get('value'), d['e2e'].get('skipped'))" 2>&1 | tail -1
done; done
