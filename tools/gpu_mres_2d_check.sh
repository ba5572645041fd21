#!/bin/bash
# Multires + solver suites after the D2Q9 multires enablement, and the sanitizer over every kernel family.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_multires.py tests/test_solver.py tests/test_capi.py tests/test_fullsize.py -q -m gpu -p no:cacheprovider > gpurun_out/m2_pytest.txt 2>&1
tail -1 gpurun_out/m2_pytest.txt; grep -E "^FAILED" gpurun_out/m2_pytest.txt | head
bash tools/gpu_sanitize.sh
