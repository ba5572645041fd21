#!/bin/bash
# Regenerate the profiles/ evidence on one B200 (run via gpurun). Tag = $1 (default r1).
# Bench lines (200 and 500 steps), the ncu launch list of bench.py, ncu --set full
# captures of the dense step, fused-probe step, block-sparse and multires kernels,
# the per-path benches and the e2e breakdown.
T=${1:-r1}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_$T.txt 2>&1
timeout 900 python bench.py --steps 500 --warmup 50 > gpurun_out/bench500_$T.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 3 -c 30 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-paths > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_step -s 3 -c 1 -o gpurun_out/dense_full_$T python tools/prof_dense.py 512 5 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_step -s 3 -c 2 -o gpurun_out/probe_full_$T python tools/prof_probe.py 512 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sparse_step -s 3 -c 2 -o gpurun_out/sparse_full_$T python tools/bench_paths.py sparse --n 512 --steps 1 --warmup 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mres_pull -s 6 -c 2 -o gpurun_out/mres_full_$T python tools/prof_mres.py 512 > /dev/null 2>&1
timeout 600 python tools/bench_paths.py sparse --n 512 --steps 20 > gpurun_out/paths_sparse_$T.txt 2>&1
timeout 600 python tools/bench_paths.py multires --n 512 --steps 5 > gpurun_out/paths_mres_$T.txt 2>&1
timeout 600 python tools/e2e_breakdown.py 512 200 > gpurun_out/e2e_$T.txt 2>&1
# ncu reports are too large to travel back: summarise them here, keep the raw
# per-launch metric pages as csv, and move the reports out of gpurun_out/
for r in gpurun_out/*_$T.ncu-rep; do
  b=${r%.ncu-rep}
  python tools/ncu_summary.py $r > $b.md 2>&1
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  mkdir -p /tmp/ncu_reps; mv $r /tmp/ncu_reps/
done
ls -la gpurun_out/*_$T*; tail -c 600 gpurun_out/bench_$T.txt; cat gpurun_out/e2e_$T.txt
cut -c1-300 gpurun_out/paths_sparse_$T.txt gpurun_out/paths_mres_$T.txt
