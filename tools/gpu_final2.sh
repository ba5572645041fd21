#!/bin/bash
# Round-end evidence, second pass: configs[0] against the reference's own
# reference_dense_run (1000 steps), the run() loop costs, then tools/gpu_final.sh.
mkdir -p gpurun_out
timeout 1500 python tools/configs0_parity.py > gpurun_out/configs0_r1.txt 2>&1; tail -1 gpurun_out/configs0_r1.txt
timeout 900 python tools/run_paths.py > gpurun_out/runpaths_r1.txt 2>&1; cat gpurun_out/runpaths_r1.txt | cut -c1-300
bash tools/gpu_final.sh r1
