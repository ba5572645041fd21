#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest9.txt 2>&1
tail -3 gpurun_out/pytest9.txt; grep -E "^FAILED|^ERROR" gpurun_out/pytest9.txt | head
