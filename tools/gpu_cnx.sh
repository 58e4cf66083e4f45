#!/bin/bash
# ConvNeXt-T / FFN: parity tests, GEMM sweep, kernel launch list, timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_convnext.py tests/test_gpu_parity.py -m gpu -x -q -k "convnext or ffn or golden or gemm" > gpurun_out/pytest_cnx.log 2>&1; echo "rc $?" >> gpurun_out/pytest_cnx.log
tail -3 gpurun_out/pytest_cnx.log
timeout 300 python tools/bench_gemm.py
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cnx_launches.csv python tools/prof_block.py cnx_stem cnx_ds1 cnx192 cnx384 cnx768 --iters 1 --timed 0 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/cnx_launches.csv')))
h=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
hd=rows[h]; k=hd.index('Kernel Name'); v=hd.index('Metric Value'); g=hd.index('Grid Size')
for r in rows[h+1:]:
    if len(r)>v and 'at::' not in r[k]: print(f"{r[k][:40]:40s} grid {r[g]:>14s} {float(r[v].replace(',',''))/1e3:9.1f} us")
PY
timeout 300 python tools/bench_convnext.py 128 224 > gpurun_out/bench_cnx.txt 2>&1
cat gpurun_out/bench_cnx.txt
