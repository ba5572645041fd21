#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -k "tolerance or multiprocess or short_run or probe" > gpurun_out/pytest_gpu2.txt 2>&1
timeout 600 python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu > gpurun_out/bench2.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:dense_step -s 2 -c 1 python tools/prof_dense.py 512 4 > gpurun_out/ncu2.txt 2>&1
tail -4 gpurun_out/pytest_gpu2.txt; tail -1 gpurun_out/bench2.txt | cut -c1-600; grep -E "duration|inst_executed|bytes|throughput" gpurun_out/ncu2.txt
