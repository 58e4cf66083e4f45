#!/bin/bash
# compute-sanitizer over the round-2 kernel paths (one small launch each)
mkdir -p gpurun_out/san
rm -f gpurun_out/san/summary_r2.txt
for c in mb_s1_7 mb_s1_14 mb_s1_s2 mb_stage cf_fused cf_wide ffn head lw_mbconv lw_convfirst; do
  for t in memcheck racecheck synccheck; do
    timeout 600 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_cases.py $c > gpurun_out/san/${c}_${t}.txt 2>&1
    echo "$c $t rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san/${c}_${t}.txt | tail -1)" >> gpurun_out/san/summary_r2.txt
  done
done
cat gpurun_out/san/summary_r2.txt
