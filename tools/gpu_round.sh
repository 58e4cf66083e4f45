# one GPU call: GPU tests, smoke, default bench, ncu launch list of a short bench,
# ncu --set full of the dominant kernels (MBConv 14x14 and stride-2 ConvFirst 112)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --skip-cpu > gpurun_out/bench_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mb_front" -s 3 -c 1 -o gpurun_out/prof_mb14 python tools/prof_block.py mb14 --iters 3 > gpurun_out/prof_mb14.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cf2_kernel" -s 3 -c 1 -o gpurun_out/prof_cfs2 python tools/prof_block.py cfs2_112 --iters 3 > gpurun_out/prof_cfs2.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; cat gpurun_out/bench.json
