#!/bin/bash
# refresh round-1 evidence for the final kernels: e2e split, path benches, ncu launch list + full captures
mkdir -p gpurun_out
timeout 600 python tools/e2e_breakdown.py 512 200 > gpurun_out/e2e19.txt 2>&1
timeout 600 python tools/bench_paths.py sparse --n 512 --steps 20 > gpurun_out/paths_sparse19.txt 2>&1
timeout 600 python tools/bench_paths.py multires --n 512 --steps 5 > gpurun_out/paths_mres19.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 3 -c 30 --csv --log-file gpurun_out/launches19.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_step -s 3 -c 1 -o gpurun_out/dense_full19 python tools/prof_dense.py 512 5 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sparse_step -s 3 -c 2 -o gpurun_out/sparse_full19 python tools/bench_paths.py sparse --n 512 --steps 1 --warmup 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mres_pull -s 6 -c 2 -o gpurun_out/mres_full19 python tools/prof_mres.py 512 > /dev/null 2>&1
ls gpurun_out/*19*; cat gpurun_out/e2e19.txt; cut -c1-300 gpurun_out/paths_sparse19.txt gpurun_out/paths_mres19.txt
