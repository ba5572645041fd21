#!/bin/bash
# ncu launch list of the default bench step loop (no paths, no e2e, no CPU leg).
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 3 -c 30 --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-paths > /dev/null 2>&1
python tools/ncu_summary.py --launches gpurun_out/launches_r1.csv
