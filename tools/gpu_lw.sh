#!/bin/bash
# layer-wise device schedules: parity tests + the fused-vs-layer-wise bench section
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layerwise.py tests/test_big_golden.py tests/test_abi.py -q -x > gpurun_out/pytest_lw.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_lw.log
timeout 600 python -c "
import json, torch, bench
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
print(json.dumps(bench.fused_vs_layer_wise(flush), indent=1))
" > gpurun_out/lw_bench.json 2> gpurun_out/lw_bench.err
tail -15 gpurun_out/pytest_lw.log; cat gpurun_out/lw_bench.json; tail -5 gpurun_out/lw_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lw_launches.csv python -c "
import torch, bench
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
bench._device_time.__defaults__ = (2, 1)
bench.fused_vs_layer_wise(flush)
" > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/lw_launches.csv 2>/dev/null | head -40
