import os, sys, time, statistics
sys.path.insert(0, "/root/repo")
import torch
import bench
from paper_2404_03617_b200.scheduler import FusedNetwork
net = bench._net("convfirstnet-pico")
m = FusedNetwork(net, batch=128, seed=1234)
gen = torch.Generator(device="cuda").manual_seed(0)
m.x.normal_(generator=gen)
g = m.capture()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
host_x = [torch.empty(m.x.shape, dtype=torch.float16, pin_memory=True) for _ in range(2)]
for hx in host_x:
    hx.copy_(m.x.cpu())
host_out = [torch.empty(m.output.shape, dtype=torch.float16, pin_memory=True) for _ in range(2)]
def e2e(steps=20, tag=""):
    m.run_host_batches([host_x[i % 2] for i in range(5)], [host_out[i % 2] for i in range(5)])
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    m.run_host_batches([host_x[i % 2] for i in range(steps)], [host_out[i % 2] for i in range(steps)])
    t1 = time.perf_counter()
    e1.record(); e1.synchronize()
    print(f"{tag:30s} e2e {e0.elapsed_time(e1)/steps:.3f} ms/step  host-issue {1e3*(t1-t0)/steps:.3f} ms/step", flush=True)
e2e(tag="fresh")
for _ in range(5): g.replay()
torch.cuda.synchronize()
for _ in range(20):
    flush.fill_(1)
    g.replay()
    torch.cuda.synchronize()
e2e(tag="after device loop")
with bench.ClockSampler(0) as clk:
    e2e(tag="with clock sampler running")
e2e(tag="after sampler")
e2e(50, tag="50 steps")
