mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -k "s2 or network or determ or full_size" 2>&1 | tail -15 > gpurun_out/pytest_cf2.log
timeout 120 python tools/prof_block.py cfs2_112 cfs2_56 > gpurun_out/unit_times_cf2.txt 2>&1
cat gpurun_out/pytest_cf2.log gpurun_out/unit_times_cf2.txt
