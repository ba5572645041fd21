#!/bin/bash
# bench.py contract test + the default bench line (with configs[3-4] paths) + the reference arm.
mkdir -p gpurun_out
T0=$(date +%s); timeout 900 python bench.py > gpurun_out/bc_bench.txt 2> gpurun_out/bc_bench.err; echo "bench wall $(( $(date +%s) - T0 )) s"
tail -1 gpurun_out/bc_bench.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['e2e']['value'], json.dumps(d['paths']))"
