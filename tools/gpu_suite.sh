#!/bin/bash
# Full GPU suite (no -x: every failure listed) + smoke. Tag = $1.
T=${1:-r2}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/suite_$T.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.txt 2>&1
tail -15 gpurun_out/suite_$T.txt; tail -2 gpurun_out/smoke_$T.txt
