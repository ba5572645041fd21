#!/bin/bash
# Multires parity suite + path bench, then the profiles/ evidence refresh.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_multires.py tests/test_solver.py tests/test_fullsize.py tests/test_capi.py -q -m gpu -p no:cacheprovider > gpurun_out/mres_pytest.txt 2>&1
tail -2 gpurun_out/mres_pytest.txt; grep -E "^FAILED|^E " gpurun_out/mres_pytest.txt | head -20
bash tools/gpu_evidence.sh r1
