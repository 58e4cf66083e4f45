"""ConvNeXt-T (BASELINE config 4) forward on one B200: CUDA-graph replays timed
with CUDA events (L2 flushed between replays), images/s, efficiency vs the
measured bf16 burst, and per-unit times. Usage: python tools/bench_convnext.py [batch] [res]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_03617_b200.convnext import convnext_tiny, network_macs, unit_macs  # noqa: E402
from paper_2404_03617_b200.scheduler import FusedNetwork  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 128
res = int(sys.argv[2]) if len(sys.argv) > 2 else 224
peaks_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
peak = json.load(open(peaks_path))["bf16_tflops"] * 1e12 if os.path.exists(peaks_path) else 1.6673e15
spec = convnext_tiny(res)
m = FusedNetwork(spec, batch=batch, seed=0)
m.x.normal_()
m.capture()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    m.replay()
torch.cuda.synchronize()
ts = []
for _ in range(20):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    m.replay()
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1) / 1e3)
ts.sort()
t = ts[len(ts) // 2]
macs = network_macs(spec)
print(json.dumps({"model": spec.name, "batch": batch, "ms": t * 1e3, "images_per_s": batch / t,
                  "tflops": 2 * macs * batch / t / 1e12, "frac_of_measured_burst": 2 * macs * batch / t / peak,
                  "launches": m.launch_count()}))
for u, inst, tu in zip(m.units, m.instances, m.time_units(10)):
    fl = 2 * unit_macs(inst) * batch
    print(f"{u.label:6s} {type(inst.block).__name__:14s} c={inst.in_channels:4d} {inst.in_h:3d}x{inst.in_w:<3d} "
          f"{tu * 1e6:8.1f} us  {fl / tu / 1e12:7.1f} TF/s")
