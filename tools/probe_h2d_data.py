"""H2D bandwidth vs buffer contents / first CPU touch (pinned, same process)."""
import torch

n = 128 * 224 * 224 * 3
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


zeros = [torch.empty(n, dtype=torch.float16, pin_memory=True) for _ in range(2)]
print(f"untouched  {bw(zeros):.1f} GB/s")
for b in zeros:
    b.zero_()
print(f"zeroed     {bw(zeros):.1f} GB/s")
rnd = [torch.empty(n, dtype=torch.float16, pin_memory=True) for _ in range(2)]
for b in rnd:
    b.copy_(torch.randn(n, dtype=torch.float32).half())
for k in range(3):
    print(f"random {k}   {bw(rnd):.1f} GB/s   zeros {bw(zeros):.1f} GB/s")
for b in zeros:
    b.copy_(rnd[0])
print(f"zeros buffers now random: {bw(zeros):.1f} GB/s")
