#!/bin/bash
# ConvNeXt-T / FFN bring-up: parity tests, kernel launch list, timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_convnext.py tests/test_gpu_parity.py -m gpu -x -q -k "convnext or ffn or golden" > gpurun_out/pytest_cnx.log 2>&1; echo "rc $?" >> gpurun_out/pytest_cnx.log
tail -5 gpurun_out/pytest_cnx.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cnx_launches.csv python tools/prof_block.py cnx_stem cnx96 cnx_ds1 cnx192 cnx384 cnx768 cnx_head --iters 1 --timed 0 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/cnx_launches.csv')))
h=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
hd=rows[h]; k=hd.index('Kernel Name'); v=hd.index('Metric Value'); g=hd.index('Grid Size'); b=hd.index('Block Size')
for r in rows[h+1:]:
    if len(r)>v: print(f"{r[k][:50]:50s} grid {r[g]:>14s} blk {r[b]:>12s} {float(r[v].replace(',',''))/1e3:9.1f} us")
PY
timeout 300 python tools/bench_convnext.py 128 224 > gpurun_out/bench_cnx.txt 2>&1
head -1 gpurun_out/bench_cnx.txt
