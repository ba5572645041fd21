#!/bin/bash
# Every GPU recipe behind profiles/, as sections of one script (run through
# gpurun on one B200; writes only under gpurun_out/):
#
#   bash tools/gpu_evidence.sh TAG [section ...]      (default: check bench ncu paths runloops e2e)
#
# Sections
#   check      full GPU suite (no -x), smoke, host / topology info
#   bench      bench.py (200 and 500 steps), the reference arm, a self-launched 2-rank bench on the one GPU
#   launches   ncu launch list (per-kernel times) of the bench step loop
#   ncu        ncu --set full of the dense step, the fused-probe step, the AoS tile step, block-sparse and
#              multires kernels, summarised on the box (tools/ncu_summary.py; reports stay in /tmp)
#   paths      per-path benches: dense layouts / lattices / precisions, block-sparse strategies, multires
#   runloops   run() loop costs (step_probe_n vs step), fused-probe overhead, clock / power-cap probe
#   e2e        where the host-API e2e time goes
#   sanitize   compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize.py
#   multirank  multi-process dense paths with ranks sharing the GPU at 512^3 (both halo modes)
#   emulate    one-rank emulation of the N-GPU strong / weak schedules (tools/emulate_rank.py)
#
# Kernel-variant sweeps (block sizes, CTA bounds, tile shapes) use
# tools/build_lib_variant.sh (here) + tools/gpu_lib_variants.sh (on the box).
T=${1:-r2}
shift
SECTIONS=${*:-check bench ncu paths runloops e2e}
mkdir -p gpurun_out /tmp/ncu_reps
ncu_capture() {  # name kernel-regex skip count cmd...
  local n=$1 k=$2 s=$3 c=$4; shift 4
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c $c -o /tmp/ncu_reps/${n}_$T "$@" > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/ncu_reps/${n}_$T.ncu-rep > gpurun_out/${n}_$T.md 2>&1
  ncu -i /tmp/ncu_reps/${n}_$T.ncu-rep --page raw --csv > gpurun_out/${n}_$T.raw.csv 2>/dev/null
}
for sec in $SECTIONS; do
  case $sec in
  check)
    (nproc; lscpu | head -20; free -g; nvidia-smi; nvidia-smi topo -m) > gpurun_out/host_$T.txt 2>&1
    timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/suite_$T.txt 2>&1
    timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.txt 2>&1
    tail -3 gpurun_out/suite_$T.txt; grep -E "^FAILED" gpurun_out/suite_$T.txt | head; tail -1 gpurun_out/smoke_$T.txt ;;
  bench)
    timeout 900 python bench.py > gpurun_out/bench_$T.txt 2>&1
    timeout 900 python bench.py --steps 500 --warmup 50 > gpurun_out/bench500_$T.txt 2>&1
    timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$T.txt 2>&1
    VOXL_SHARE_DEVICE=1 timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench2_$T.txt 2>&1
    tail -c 1200 gpurun_out/bench_$T.txt; echo; tail -c 400 gpurun_out/bench_ref_$T.txt; echo ;;
  launches)
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 3 -c 30 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-paths > /dev/null 2>&1
    python tools/ncu_summary.py --launches gpurun_out/launches_$T.csv | tail -12 ;;
  ncu)
    ncu_capture dense_step dense_step 3 1 python tools/prof_dense.py 512 5
    ncu_capture dense_probe dense_step 2 2 python tools/prof_probe.py 512
    ncu_capture dense_aos aos_tiled 2 1 python tools/prof_aos.py
    ncu_capture sparse sparse_step 3 2 python tools/bench_paths.py sparse --n 512 --steps 1 --warmup 0
    ncu_capture mres mres_pull 6 2 python tools/prof_mres.py 512
    for f in gpurun_out/*_$T.md; do head -8 $f; done ;;
  paths)
    timeout 900 python tools/bench_paths.py dense --n 512 --steps 20 > gpurun_out/paths_dense_$T.txt 2>&1
    timeout 600 python tools/bench_paths.py sparse --n 512 --steps 20 > gpurun_out/paths_sparse_$T.txt 2>&1
    timeout 600 python tools/bench_paths.py multires --n 512 --steps 5 > gpurun_out/paths_mres_$T.txt 2>&1
    timeout 900 python tools/bench_paths.py sparse --n 512 --steps 20 --lattice D3Q27 > gpurun_out/paths_sparse27_$T.txt 2>&1
    cut -c1-260 gpurun_out/paths_*_$T.txt ;;
  runloops)
    timeout 900 python tools/run_paths.py --n 512 --steps 200 > gpurun_out/run_paths_$T.txt 2>&1
    timeout 600 python tools/probe_overhead.py > gpurun_out/probe_overhead_$T.txt 2>&1
    timeout 600 python tools/clock_probe.py > gpurun_out/clock_probe_$T.txt 2>&1
    cat gpurun_out/run_paths_$T.txt gpurun_out/probe_overhead_$T.txt ;;
  e2e)
    timeout 600 python tools/e2e_breakdown.py 512 200 > gpurun_out/e2e_$T.txt 2>&1; cat gpurun_out/e2e_$T.txt ;;
  sanitize)
    for tool in memcheck racecheck synccheck; do
      timeout 1800 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize.py > gpurun_out/san_${tool}_$T.txt 2>&1
      echo "$tool rc=$?"; grep -E "ERROR SUMMARY|sanitize run ok" gpurun_out/san_${tool}_$T.txt | head -3
    done ;;
  multirank)
    for n in 2 4 8; do for h in zero_copy copy; do
      VOXL_SHARE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --steps 10 --warmup 3 --no-cpu --halo $h > gpurun_out/multirank_${n}_${h}_$T.txt 2>&1
      echo "N=$n $h rc=$?"; tail -1 gpurun_out/multirank_${n}_${h}_$T.txt | cut -c1-300
    done; done ;;
  emulate)
    timeout 600 python tools/emulate_rank.py > gpurun_out/emulate_strong_$T.txt 2>&1
    timeout 900 python tools/emulate_rank.py --weak > gpurun_out/emulate_weak_$T.txt 2>&1
    tail -1 gpurun_out/emulate_strong_$T.txt; tail -1 gpurun_out/emulate_weak_$T.txt ;;
  *) echo "unknown section $sec" ;;
  esac
done
