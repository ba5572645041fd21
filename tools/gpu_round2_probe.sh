mkdir -p gpurun_out
(nproc; lscpu | head -20; free -g; nvidia-smi; nvidia-smi topo -m) > gpurun_out/g1_host.txt 2>&1
timeout 300 ./tools/micro/host_io 4 > gpurun_out/g1_hostio4.txt 2>&1
timeout 300 ./tools/micro/host_io 16 > gpurun_out/g1_hostio16.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g1_suite.txt 2>&1
tail -3 gpurun_out/g1_suite.txt; cat gpurun_out/g1_hostio*.txt
