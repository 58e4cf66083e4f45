mkdir -p gpurun_out
for m in convfirstnet-pico convfirstnet-nano convfirstnet-tiny convfirstnet-small; do
  timeout 600 python bench.py --model $m --skip-configs --skip-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$m', round(d['value']), round(d['e2e']['value']), round(d['efficiency']['tflops'],1), round(d['efficiency']['frac_of_measured_burst'],4))"
done > gpurun_out/zoo.txt 2>&1
cat gpurun_out/zoo.txt
