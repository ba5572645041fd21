#!/bin/bash
# One ncu --set full capture summarised on the box (reports are too large to
# travel): gpu_ncu.sh TAG KERNEL_REGEX SKIP COUNT cmd...  -> gpurun_out/TAG.md + TAG.raw.csv
T=$1; K=$2; S=$3; C=$4; shift 4
mkdir -p gpurun_out /tmp/ncu_reps
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c $C -o /tmp/ncu_reps/$T "$@" > gpurun_out/$T.log 2>&1
python tools/ncu_summary.py /tmp/ncu_reps/$T.ncu-rep > gpurun_out/$T.md 2>&1
ncu -i /tmp/ncu_reps/$T.ncu-rep --page raw --csv > gpurun_out/$T.raw.csv 2>/dev/null
ncu -i /tmp/ncu_reps/$T.ncu-rep --page source --csv > gpurun_out/$T.source.csv 2>/dev/null
head -c 3000 gpurun_out/$T.md
