#!/bin/bash
# ncu --set full of the network-front kernels (first launch of each) in a short bench run
mkdir -p gpurun_out
for k in stem_cf cf2_kernel mb_front_kernel cf_fused_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 0 -c 1 -o gpurun_out/ncu_$k python bench.py --steps 1 --warmup 3 --skip-cpu --skip-configs > /dev/null 2>&1
done
ls -la gpurun_out/*.ncu-rep | tail -4
