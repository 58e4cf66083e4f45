"""H2D bandwidth of pinned host buffers allocated with the process bound to
each NUMA node's CPUs (first-touch places the pinned pages on that node), plus
the GPU's own NUMA node from sysfs. One subprocess per node."""
import glob
import os
import subprocess
import sys

N = 128 * 224 * 224 * 3


def measure():
    import torch

    bufs = [torch.empty(N, dtype=torch.float16, pin_memory=True) for _ in range(2)]
    for b in bufs:
        b.fill_(1.0)
    dev = torch.empty(N, dtype=torch.float16, device="cuda")
    for _ in range(3):
        for b in bufs:
            dev.copy_(b, non_blocking=True)
    torch.cuda.synchronize()
    out = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(40):
            dev.copy_(bufs[i % 2], non_blocking=True)
        e1.record()
        e1.synchronize()
        out.append(N * 2 * 40 / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return out


def cpulist(text):
    cpus = set()
    for part in text.strip().split(","):
        if "-" in part:
            a, b = part.split("-")
            cpus.update(range(int(a), int(b) + 1))
        elif part:
            cpus.add(int(part))
    return cpus


if __name__ == "__main__":
    if len(sys.argv) > 1:
        cpus = cpulist(sys.argv[1])
        os.sched_setaffinity(0, cpus)
        print(" ".join(f"{v:.1f}" for v in measure()))
        sys.exit(0)
    import torch

    p = torch.cuda.get_device_properties(0)
    bdf = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    print("gpu", bdf)
    for f in ("numa_node", "local_cpulist"):
        try:
            print(f, open(f"/sys/bus/pci/devices/{bdf}/{f}").read().strip())
        except OSError as e:
            print(f, "n/a", e)
    print("allowed cpus", len(os.sched_getaffinity(0)))
    for node in sorted(glob.glob("/sys/devices/system/node/node[0-9]*")):
        cl = open(f"{node}/cpulist").read().strip()
        allowed = cpulist(cl) & os.sched_getaffinity(0)
        if not allowed:
            print(os.path.basename(node), cl, "no allowed cpus")
            continue
        r = subprocess.run([sys.executable, __file__, ",".join(map(str, sorted(allowed)))], capture_output=True,
                           text=True, timeout=300)
        print(os.path.basename(node), cl, "H2D GB/s:", r.stdout.strip(), r.stderr.strip()[-200:])
    r = subprocess.run([sys.executable, __file__, ",".join(map(str, sorted(os.sched_getaffinity(0))))],
                       capture_output=True, text=True, timeout=300)
    print("unbound H2D GB/s:", r.stdout.strip())
