#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest28.txt 2>&1
timeout 600 python tools/e2e_breakdown.py 512 200 > gpurun_out/e2e28.txt 2>&1
tail -2 gpurun_out/pytest28.txt; grep -E "^FAILED|^E " gpurun_out/pytest28.txt | head; cat gpurun_out/e2e28.txt
