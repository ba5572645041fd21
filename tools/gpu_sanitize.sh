#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize.py (small runs of every kernel family).
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1800 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize.py > gpurun_out/san_$tool.txt 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|sanitize run ok|Error" gpurun_out/san_$tool.txt | head -5
done
