#!/bin/bash
# round-2 evidence: GPU tests, smoke, default bench (+ other configs), launch list of a short bench,
# ncu --set full of the dominant kernel (the 14x14 MBConv stage launch) and of the fused stem + s1b0
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --skip-cpu --skip-configs > gpurun_out/bench_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mb_s1 -s 3 -c 1 -o gpurun_out/ncu_stage14 python bench.py --steps 1 --warmup 3 --skip-cpu --skip-configs > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stem_cf -s 1 -c 1 -o gpurun_out/ncu_stem_cf python bench.py --steps 1 --warmup 3 --skip-cpu --skip-configs > /dev/null 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
