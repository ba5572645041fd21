#!/bin/bash
# Stall-guard test, emulated rank scaling, and the fused-probe partial variants timed on one B200.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_multigpu.py -q -m gpu -p no:cacheprovider -k stalled > gpurun_out/stall_pytest.txt 2>&1
tail -2 gpurun_out/stall_pytest.txt; grep -E "^E " gpurun_out/stall_pytest.txt | head -5
timeout 600 python tools/emulate_rank.py > gpurun_out/emulate.txt 2>&1; tail -2 gpurun_out/emulate.txt
bash tools/build_variants.sh > gpurun_out/variants_build.txt 2>&1
cp paper_2503_07898_b200/_lib/libvoxl_b200.so /tmp/libvoxl_b200.so.orig
for t in w1 w0 w1 w0; do
  cp _libvar/$t/libvoxl_b200.so paper_2503_07898_b200/_lib/libvoxl_b200.so
  TAG=$t timeout 300 python tools/time_probe.py 512 100 >> gpurun_out/probe_variants.txt 2>&1
done
cp /tmp/libvoxl_b200.so.orig paper_2503_07898_b200/_lib/libvoxl_b200.so
cat gpurun_out/probe_variants.txt
