#!/bin/bash
# Both bench arms with the resident reference loop, and the C-ABI / drop-in tests.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_capi.py tests/test_oracle.py -q -m "gpu or not gpu" -p no:cacheprovider > gpurun_out/cl_pytest.txt 2>&1; tail -1 gpurun_out/cl_pytest.txt; grep -E "^FAILED" gpurun_out/cl_pytest.txt | head
timeout 900 python bench.py --impl reference > gpurun_out/cl_ref.txt 2>&1; tail -1 gpurun_out/cl_ref.txt | cut -c1-200; tail -1 gpurun_out/cl_ref.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['cpu_baseline'])"
timeout 900 python bench.py > gpurun_out/cl_bench.txt 2>&1; tail -1 gpurun_out/cl_bench.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['cpu_baseline'])"
