#!/bin/bash
# compute-sanitizer pass over one small launch per kernel family + MBConv phase traces
mkdir -p gpurun_out/san
timeout 300 python tools/trace_mb1.py 14 7 > gpurun_out/trace_mb1.txt 2>&1
for c in cf_fused cf_convnext cf_s2 mb_s1_14 mb_s1_7 mb_front_pair mb_front_s2 mb_front_t1 stem head; do
  for t in memcheck racecheck synccheck initcheck; do
    timeout 600 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_cases.py $c > gpurun_out/san/${c}_${t}.txt 2>&1
    echo "$c $t rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san/${c}_${t}.txt | tail -1)" >> gpurun_out/san/summary.txt
  done
done
cat gpurun_out/trace_mb1.txt gpurun_out/san/summary.txt
