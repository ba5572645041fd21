#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest31.txt 2>&1
tail -2 gpurun_out/pytest31.txt; grep -E "^FAILED|^E " gpurun_out/pytest31.txt | head -20
