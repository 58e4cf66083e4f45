mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
python tools/prof_block.py mb14 mb7 mbs2_28 mbs2_14 > gpurun_out/unit_times.txt 2>&1
cat gpurun_out/pytest_gpu.log; cat gpurun_out/unit_times.txt
