#!/bin/bash
# Final-commit verification: full GPU suite, smoke, default bench line, run() loop costs, sanitizer.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/last2_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/last2_pytest.txt
tail -2 gpurun_out/last2_pytest.txt; grep -E "^FAILED" gpurun_out/last2_pytest.txt | head
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/last2_bench.txt 2>&1; tail -1 gpurun_out/last2_bench.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'], json.dumps(d['paths'])[:300])"
timeout 900 python tools/run_paths.py > gpurun_out/last2_runpaths.txt 2>&1; cut -c1-200 gpurun_out/last2_runpaths.txt
bash tools/gpu_sanitize.sh
