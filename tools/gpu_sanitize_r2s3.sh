#!/bin/bash
# compute-sanitizer over the kernels changed in round 2 session 3 (one small launch each)
mkdir -p gpurun_out/san
rm -f gpurun_out/san/summary_r2s3.txt
for c in cf_s2 cf_fused mb_s1_14 mb_s1_7 mb_stage mb_front_s2 mb_front_t1 ffn cnx_c192 cnx_c384 cnx_c96_big; do
  for t in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_cases.py $c > gpurun_out/san/${c}_${t}.txt 2>&1
    echo "$c $t rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san/${c}_${t}.txt | tail -1)" >> gpurun_out/san/summary_r2s3.txt
  done
done
cat gpurun_out/san/summary_r2s3.txt
