#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke7.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu7.txt 2>&1
timeout 900 python bench.py --steps 100 --warmup 10 > gpurun_out/bench7.txt 2>&1
timeout 600 python tools/bench_paths.py sparse --n 512 --steps 20 > gpurun_out/paths_sparse7.txt 2>&1
timeout 600 python tools/bench_paths.py multires --n 512 --steps 5 > gpurun_out/paths_mres7.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_dense.csv python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_step -s 2 -c 1 -o gpurun_out/dense_full7 python tools/prof_dense.py 512 4 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sparse_step -s 3 -c 2 -o gpurun_out/sparse_full7 python tools/bench_paths.py sparse --n 256 --steps 1 --warmup 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mres_pull -s 6 -c 2 -o gpurun_out/mres_full7 python tools/prof_mres.py 256 > /dev/null 2>&1
tail -3 gpurun_out/pytest_gpu7.txt; cut -c1-300 gpurun_out/bench7.txt; cut -c1-250 gpurun_out/paths_sparse7.txt gpurun_out/paths_mres7.txt
