#!/bin/bash
# Run CMD once per prebuilt _libvar/*/libvoxl_b200.so (and the in-tree build as "base"), twice round-robin.
# Usage: gpu_lib_variants.sh TAG "CMD"   (VOXL_TAG names the variant inside CMD's output)
T=$1; CMD=$2
mkdir -p gpurun_out
L=paper_2503_07898_b200/_lib/libvoxl_b200.so
cp $L /tmp/base.so
for r in 1 2; do
  for d in base _libvar/*/; do
    if [ "$d" = base ]; then cp /tmp/base.so $L; n=base; else cp $d/libvoxl_b200.so $L; n=$(basename $d); fi
    VOXL_TAG=$n bash -c "$CMD" >> gpurun_out/variants_$T.txt 2>&1
  done
done
cp /tmp/base.so $L
cat gpurun_out/variants_$T.txt
