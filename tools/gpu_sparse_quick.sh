#!/bin/bash
# Block-sparse parity suite (twice: the step uses two streams) + the 512^3 sparse path bench (D3Q19, D3Q27).
mkdir -p gpurun_out
for i in 1 2; do
timeout 1500 python -m pytest tests/test_sparse.py tests/test_solver.py tests/test_fullsize.py tests/test_capi.py tests/test_tolerance_large.py -q -m gpu -p no:cacheprovider -k "not mres and not multires" > gpurun_out/sq_pytest_$i.txt 2>&1
tail -1 gpurun_out/sq_pytest_$i.txt; grep -E "^FAILED|^E " gpurun_out/sq_pytest_$i.txt | head -20
done
timeout 600 python tools/bench_paths.py sparse --n 512 --steps 20 > gpurun_out/sq_paths.txt 2>&1
timeout 600 python tools/bench_paths.py sparse --n 512 --steps 10 --lattice D3Q27 > gpurun_out/sq_paths27.txt 2>&1
python - <<'PY'
import json
for f in ("gpurun_out/sq_paths.txt", "gpurun_out/sq_paths27.txt"):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l); print(d["lattice"], d["strategy"], d["MLUPS"], d["frac_of_measured_peak"], d["boundary_kernel_ms"], d["light_kernel_ms"])
        else: print(l.rstrip()[:300])
PY
