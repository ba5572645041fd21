#!/bin/bash
# Multires parity suite three times over (the fused schedule uses two streams).
mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 900 python -m pytest tests/test_multires.py tests/test_fullsize.py tests/test_tolerance_large.py -q -m gpu -p no:cacheprovider -k "mres or multires or fused or Mres" > gpurun_out/mr_$i.txt 2>&1
  tail -1 gpurun_out/mr_$i.txt; grep -E "^FAILED" gpurun_out/mr_$i.txt | head
done
