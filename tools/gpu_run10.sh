#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu > gpurun_out/bench10.txt 2>&1
timeout 900 python -m pytest tests/test_dense_gpu.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest10.txt 2>&1
tail -2 gpurun_out/pytest10.txt; python -c "
import json; d=json.loads(open('gpurun_out/bench10.txt').read().strip().splitlines()[-1]); print(d['value'], d['roofline'], d['clocks'])"
