"""BASELINE config 5 on one B200: batch sweep 128..1024 of ConvFirstNet-Pico and
ConvNeXt-T (CUDA graphs, device-resident inputs, L2 flushed per replay),
written as gap samples (reference CSV schema) and the efficiency-gap plot on
the b200-measured device. Usage: python tools/gap_sweep.py [outdir]"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_03617_b200 import complexity, gap, zoo  # noqa: E402
from paper_2404_03617_b200.convnext import convnext_tiny, network_macs  # noqa: E402
from paper_2404_03617_b200.scheduler import FusedNetwork  # noqa: E402

out_dir = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
os.makedirs(out_dir, exist_ok=True)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
# accuracy: the paper's ImageNet top-1 (reference data/model_speed_accuracy.csv);
# these are random-init weights, so only latency is measured here
models = [("convfirst-pico@224", lambda: zoo.at_resolution(zoo.from_name("convfirstnet-pico"), 224), 79.9),
          ("convnext-tiny@224", lambda: convnext_tiny(224), 82.1)]
samples = []
for name, mk, acc in models:
    net = mk()
    macs = network_macs(net) if hasattr(net, "plan") else complexity.network_macs(net)
    for batch in (128, 256, 512, 1024):
        m = FusedNetwork(net, batch=batch, seed=1)
        m.x.normal_()
        m.capture()
        for _ in range(3):
            m.replay()
        ts = []
        for _ in range(8):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            m.replay()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        t = statistics.median(ts)
        samples.append(gap.MeasuredSample(name, macs, batch, t, acc))
        print(f"{name} b{batch}: {t * 1e3:.3f} ms  {batch / t:.0f} img/s", flush=True)
        del m
        torch.cuda.empty_cache()
dev = gap.load_device("b200-measured")
gap.write_samples_csv(os.path.join(out_dir, "gap_samples_b200.csv"), samples)
pts = gap.gap_series(samples, dev)
for p in pts:
    print(f"{p.sample.model} b{p.sample.batch}: efficiency {100 * p.efficiency:.1f}%  gap {p.gap_width:.2f}")
with open(os.path.join(out_dir, "gap_plot_b200.svg"), "w") as fh:
    fh.write(gap.gap_plot(pts, dev, "Efficiency gap on B200 (measured peak), batch 128-1024"))
