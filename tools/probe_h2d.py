"""Pinned host->device copy bandwidth of one batch (38.5 MB, Pico b128 input):
one copy vs the batch split over several streams."""
import torch

n = 128 * 224 * 224 * 3
host = torch.empty(n, dtype=torch.float16, pin_memory=True)
dev = torch.empty(n, dtype=torch.float16, device="cuda")
for parts in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(parts)]
    chunk = (n + parts - 1) // parts
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k, s in enumerate(streams):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                dev[k * chunk:(k + 1) * chunk].copy_(host[k * chunk:(k + 1) * chunk], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        e1.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"parts {parts}: {ms:.3f} ms  {n * 2 / ms / 1e6:.1f} GB/s")
