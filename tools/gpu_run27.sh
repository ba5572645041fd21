#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench27.txt 2>&1
timeout 900 python bench.py --steps 500 --warmup 50 > gpurun_out/bench27_500.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_step -s 3 -c 2 -o gpurun_out/probe_full27 python tools/prof_probe.py 512 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/probe27.csv python tools/prof_probe.py 512 > /dev/null 2>&1
timeout 600 python tools/e2e_breakdown.py 512 200 > gpurun_out/e2e27.txt 2>&1
tail -1 gpurun_out/bench27.txt | cut -c1-200; for f in gpurun_out/bench27.txt gpurun_out/bench27_500.txt; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"; done; cat gpurun_out/e2e27.txt
