#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum --clock-control none -k regex:mres_fused -s 4 -c 2 python tools/prof_mres.py 256 > gpurun_out/ncu_mres.txt 2>&1
grep -E "mres_fused|dram__|duration|inst_exec|sectors|requests|warps_active|sm__throughput|registers" gpurun_out/ncu_mres.txt | sed 's/  */ /g' | cut -c1-140
