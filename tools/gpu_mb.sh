mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "mbconv or network or device or determ or full_size or golden" 2>&1 | tail -15 > gpurun_out/pytest_mb.log
python tools/trace_mb.py mb14 mb7 mbs2 > gpurun_out/trace_mb.txt 2>&1
python tools/prof_block.py mb14 mb7 mbs2_28 mbs2_14 > gpurun_out/unit_times.txt 2>&1
cat gpurun_out/pytest_mb.log; grep -v chunk gpurun_out/trace_mb.txt; cat gpurun_out/unit_times.txt
