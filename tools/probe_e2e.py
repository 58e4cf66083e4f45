"""Where the end-to-end (host batches) time goes for Pico b128: forwards alone,
copies alone, forwards with independent concurrent copies, run_host_batches."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_03617_b200 import zoo  # noqa: E402
from paper_2404_03617_b200.scheduler import FusedNetwork  # noqa: E402


def timed(fn, steps):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn(steps)
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / steps


net = zoo.at_resolution(zoo.from_name("convfirstnet-pico"), 224)
m = FusedNetwork(net, batch=128, seed=1)
m.x.normal_()
g = m.capture()
host = [torch.empty(m.x.shape, dtype=torch.float16, pin_memory=True) for _ in range(2)]
outs = [torch.empty(m.output.shape, dtype=torch.float16, pin_memory=True) for _ in range(2)]
if "--real" in sys.argv:
    for h in host:
        h.copy_(m.x.cpu())
dev2 = torch.empty_like(m.x)
cs = torch.cuda.Stream()


def fwd(n):
    for _ in range(n):
        g.replay()


def copies(n):
    with torch.cuda.stream(cs):
        for i in range(n):
            dev2.copy_(host[i % 2], non_blocking=True)
    torch.cuda.current_stream().wait_stream(cs)


def both(n):
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs):
        for i in range(n):
            dev2.copy_(host[i % 2], non_blocking=True)
    for _ in range(n):
        g.replay()
    torch.cuda.current_stream().wait_stream(cs)


def e2e(n):
    m.run_host_batches([host[i % 2] for i in range(n)], [outs[i % 2] for i in range(n)])


for f in (fwd, copies, both, e2e, fwd, e2e):
    f(3)
    print(f"{f.__name__:8s} {timed(f, 20):.3f} ms/step")
