#!/bin/bash
# Full GPU suite (prints of the large tolerance runs kept) + smoke on one B200.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total --format=csv,noheader > gpurun_out/suite_gpu.txt; free -g >> gpurun_out/suite_gpu.txt
timeout 600 python -m pytest tests/test_tolerance_large.py -q -s -m gpu -p no:cacheprovider > gpurun_out/suite_tol.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --deselect tests/test_tolerance_large.py > gpurun_out/suite_pytest.txt 2>&1
echo "rc=$?" >> gpurun_out/suite_pytest.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/suite_smoke.txt 2>&1
cat gpurun_out/suite_gpu.txt; grep -E "max rel|passed|failed|^E " gpurun_out/suite_tol.txt | head; tail -3 gpurun_out/suite_pytest.txt; grep -E "^FAILED|^E " gpurun_out/suite_pytest.txt | head; tail -2 gpurun_out/suite_smoke.txt
