"""H2D bandwidth of pinned buffers allocated early (process start) vs late
(after the model, its graph and the device-timed loop), same process."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2404_03617_b200.scheduler import FusedNetwork  # noqa: E402

n = 128 * 224 * 224 * 3
early = [torch.empty(n, dtype=torch.float16, pin_memory=True) for _ in range(2)]
dev = torch.empty(n, dtype=torch.float16, device="cuda")


def bw(bufs, reps=40):
    for b in bufs:
        dev.copy_(b, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps):
        dev.copy_(bufs[i % 2], non_blocking=True)
    e1.record()
    e1.synchronize()
    return n * 2 * reps / (e0.elapsed_time(e1) / 1e3) / 1e9


print(f"early, at start: {bw(early):.1f} GB/s")
m = FusedNetwork(bench._net("convfirstnet-pico"), batch=128, seed=1)
m.x.normal_()
g = m.capture()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(20):
    flush.fill_(1)
    g.replay()
torch.cuda.synchronize()
late = [torch.empty(n, dtype=torch.float16, pin_memory=True) for _ in range(2)]
for b in late:
    b.copy_(m.x.reshape(-1).cpu())
for k in range(3):
    print(f"round {k}: early {bw(early):.1f} GB/s   late {bw(late):.1f} GB/s")

# the same late buffers copied as two halves on two streams (two copy engines)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def bw2(bufs, reps=40):
    half = n // 2
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in (s1, s2):
        s.wait_event(e0)
    for i in range(reps):
        with torch.cuda.stream(s1):
            dev[:half].copy_(bufs[i % 2][:half], non_blocking=True)
        with torch.cuda.stream(s2):
            dev[half:].copy_(bufs[i % 2][half:], non_blocking=True)
    for s in (s1, s2):
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    e1.synchronize()
    return n * 2 * reps / (e0.elapsed_time(e1) / 1e3) / 1e9


for k in range(3):
    print(f"two streams {k}: early {bw2(early):.1f} GB/s   late {bw2(late):.1f} GB/s   late 1-stream {bw(late):.1f}")
