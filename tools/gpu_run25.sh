#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/e2e_breakdown.py 512 200 > gpurun_out/e2e25.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest25.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench25.txt 2>&1
tail -2 gpurun_out/pytest25.txt; grep -E "^FAILED|^E " gpurun_out/pytest25.txt | head; cat gpurun_out/e2e25.txt; tail -1 gpurun_out/bench25.txt | cut -c1-300; tail -1 gpurun_out/bench25.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['e2e'])"
