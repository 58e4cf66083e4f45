"""Measured waterline of a whole network on one B200 (the paper's waterline
and efficiency-gap analysis with measured per-unit latencies).

For every plan_blocks unit: its BLOCK_FUSION workload (complexity/expand_network
accounting: ops and DRAM bytes), the attainable latency on a B200 DeviceSpec
(perf.attainable_latency: min over the tensor and HBM roofs), the measured
latency (CUDA events, FusedNetwork.time_units) and the fraction of the roof
reached. Then the network's waterline verdict (perf.waterline) against the
measured sum. Usage: python tools/waterline_report.py [model] [batch]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_03617_b200 import complexity, perf, zoo  # noqa: E402
from paper_2404_03617_b200.core import DeviceSpec, ExecutionScheme, KernelWorkload  # noqa: E402
from paper_2404_03617_b200.scheduler import FusedNetwork  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "convfirstnet-pico"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 128
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peaks = {}
try:
    peaks = json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))
except OSError:
    pass
tf = float(peaks.get("bf16_tflops", 1643.3)) * 1e12
bw = float(peaks.get("hbm_gbs", 6535.1)) * 1e9
dev = DeviceSpec("b200-measured", tf, bw, bytes_per_element=2)
net = zoo.at_resolution(zoo.from_name(model), 224)
m = FusedNetwork(net, batch=batch, seed=0)
m.x.normal_()
times = m.time_units(iters=20)
work = []  # one workload per launched unit (a fused block; stem / head summed over their layers)
for inst in m.instances:
    c = complexity.block_costs(inst.block, inst.dims(batch), ExecutionScheme.BLOCK_FUSION, dev,
                               out_channels=inst.out_channels)
    cs = c if isinstance(c, list) else [c]
    work.append(KernelWorkload(inst.label, sum(x.ops for x in cs), sum(x.bytes for x in cs), inst.dims(batch)))
rows = perf.measured_waterline(work, times, dev)
wl = perf.waterline(work, dev)
print(f"# {model}@224 b{batch} on one B200; roofs: {tf/1e12:.0f} TFLOP/s tensor, {bw/1e9:.0f} GB/s HBM (MEASURED_PEAKS.json)")
print(f"# {'unit':32s} {'bound':7s} {'GFLOP':>8s} {'MB':>8s} {'attain us':>10s} {'meas us':>9s} {'of roof':>8s} {'TFLOP/s':>8s}")
for u, r in zip(m.units, rows):
    print(f"  {u.label:6s} {type(u.block).__name__[:25]:25s} {r.bound.name.lower():7s} {r.ops/1e9:8.2f} {r.bytes/1e6:8.1f} "
          f"{r.attainable_s*1e6:10.1f} {r.measured_s*1e6:9.1f} {100*r.efficiency:7.1f}% {r.tflops:8.1f}")
tot_m = sum(times)
print(f"# network: attainable (waterline) {wl.total_latency*1e6:.1f} us, measured {tot_m*1e6:.1f} us "
      f"-> {100*wl.total_latency/tot_m:.1f}% of the waterline; computational efficiency "
      f"{sum(r.ops for r in rows)/tot_m/tf*100:.1f}% of the tensor roof")
