#!/bin/bash
# Round-end evidence on one B200: full GPU suite + smoke, both bench arms,
# ncu captures (tools/gpu_evidence.sh), emulated multi-GPU scaling (strong, weak).
T=${1:-r1}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/final_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/final_pytest.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.txt 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/final_bench_ref.txt 2>&1
bash tools/gpu_evidence.sh $T > gpurun_out/final_evidence.txt 2>&1
timeout 600 python tools/emulate_rank.py > gpurun_out/emulate_strong_$T.txt 2>&1
timeout 900 python tools/emulate_rank.py --weak > gpurun_out/emulate_weak_$T.txt 2>&1
tail -3 gpurun_out/final_pytest.txt; grep -E "^FAILED" gpurun_out/final_pytest.txt | head; tail -1 gpurun_out/final_smoke.txt
tail -1 gpurun_out/final_bench_ref.txt | cut -c1-300
tail -1 gpurun_out/bench_$T.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline'], d['e2e']['value'], json.dumps(d['paths']))"
tail -1 gpurun_out/emulate_strong_$T.txt; tail -1 gpurun_out/emulate_weak_$T.txt
