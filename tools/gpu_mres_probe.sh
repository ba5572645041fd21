#!/bin/bash
# Multires pull-probe: parity suites (run() diagnostics vs the reference) + the run() loop cost.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_multires.py tests/test_solver.py tests/test_capi.py tests/test_fullsize.py -q -m gpu -p no:cacheprovider > gpurun_out/mp_pytest.txt 2>&1
tail -1 gpurun_out/mp_pytest.txt; grep -E "^FAILED|^E " gpurun_out/mp_pytest.txt | head -10
timeout 900 python tools/run_paths.py > gpurun_out/mp_runpaths.txt 2>&1; cut -c1-250 gpurun_out/mp_runpaths.txt
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python -c "
import paper_2503_07898_b200 as V
for lat, dom in (('D3Q19', (32,32,32)), ('D2Q9', (32,48,1))):
    for prec in ('fp32', 'fp64'):
        e = V.MultiResEngine(dom, 3, level_map=V.band_level_map(dom, 3, axis=2 if dom[2] > 1 else 1), fused=True, precision=prec, lattice=lat)
        e.step(2); d = e.probe(); e.close()
print('ok')
" 2>&1 | tail -3
