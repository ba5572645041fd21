#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest17.txt 2>&1
timeout 600 python tools/e2e_breakdown.py 512 200 > gpurun_out/e2e17.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench17.txt 2>&1
tail -3 gpurun_out/pytest17.txt; grep -E "^FAILED|Error" gpurun_out/pytest17.txt | head; tail -1 gpurun_out/e2e17.txt; tail -1 gpurun_out/bench17.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'], d['roofline']['frac'])"
