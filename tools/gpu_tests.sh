#!/bin/bash
# Selected GPU test files (no -x), then optional extra commands from $EXTRA. Usage: gpu_tests.sh TAG file1 [file2 ...]
T=$1; shift
mkdir -p gpurun_out
timeout 2400 python -m pytest "$@" -m gpu -q -p no:cacheprovider > gpurun_out/tests_$T.txt 2>&1
tail -25 gpurun_out/tests_$T.txt
if [ -n "$EXTRA" ]; then bash -c "$EXTRA"; fi
