#!/bin/bash
# Round-end style check on one B200: full GPU suite, smoke, both bench arms.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > gpurun_out/full_gpu.txt
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/full_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/full_pytest.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/full_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/full_bench.txt 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/full_bench_ref.txt 2>&1
tail -3 gpurun_out/full_pytest.txt; grep -E "^FAILED|^E " gpurun_out/full_pytest.txt | head -20
tail -2 gpurun_out/full_smoke.txt; tail -c 1500 gpurun_out/full_bench.txt; tail -c 800 gpurun_out/full_bench_ref.txt
