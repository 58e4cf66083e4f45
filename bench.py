"""Benchmark: ConvFirstNet @224, batch 128 per GPU, fp16 inference through the
fused sm_100a block kernels (BASELINE.json: images/sec and computational
efficiency = 2 MACs B / t / R_peak).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--model NAME] [--impl ours|reference]

N > 1 runs under torchrun (one process per GPU, NCCL only for the barrier and
the max-over-ranks of the step time): every rank processes an independent
128-image shard (weak scaling; no collective on the data path).
``--impl reference`` times the CPU oracle port of the reference algorithm on
the host cores (rank 0 only) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

PEAK_DATASHEET = 2.25e15


def _peaks():
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["bf16_tflops"]) * 1e12, float(d["bf16_tflops_sustained"]) * 1e12, float(d["hbm_gbs"]) * 1e9, "measured"
    except Exception:
        return 1.59e15, 1.4e15, 6.65e12, "fallback"


def _net(name: str):
    from paper_2404_03617_b200 import zoo

    return zoo.at_resolution(zoo.from_name(name), 224)


# --------------------------------------------------------------- CPU arm


def cpu_sample(model: str, images: int = 1, seed: int = 0):
    """Time the CPU oracle (numpy restatement of the reference path) on
    ``images`` images of the workload. Returns (seconds, images, threads)."""
    import numpy as np

    from oracle import model as om
    from paper_2404_03617_b200.blocks import init_weights
    from paper_2404_03617_b200.core import plan_blocks
    from paper_2404_03617_b200.machine import build_schedule

    net = _net(model)
    units = plan_blocks(net)
    weights = {}
    for i, u in enumerate(units):
        s = build_schedule(u.block, u.dims(images), out_channels=u.out_channels)
        weights[u.label] = init_weights(s, np.random.default_rng(seed + i))
    x = np.random.default_rng(seed).standard_normal((images, 224, 224, 3)).astype(np.float16).astype(np.float32)
    threads = 1
    try:
        from threadpoolctl import threadpool_info

        threads = max([p.get("num_threads", 1) for p in threadpool_info()] + [1])
    except Exception:
        pass
    t0 = time.perf_counter()
    om.network_forward(units, weights, x)
    return time.perf_counter() - t0, images, threads


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    times = []
    for _ in range(args.warmup if args.warmup < 1 else 1):
        cpu_sample(args.model, 1)
    threads = 1
    for _ in range(args.steps):
        t, imgs, threads = cpu_sample(args.model, 1)
        times.append(t / imgs)
    per_img = statistics.mean(times)
    from paper_2404_03617_b200 import complexity

    macs = complexity.network_macs(_net(args.model))
    v = 1.0 / per_img
    line = {
        "impl": "reference",
        "metric": f"images/sec ({args.model}@224 inference)",
        "value": v,
        "unit": "images/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": per_img * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "fp32 storage / fp64 accumulate (reference tensor-machine numerics)",
        "data": "synthetic (fan-in scaled random-init weights, N(0,1) images)",
        "config": {"workload": f"{args.model}@224 forward, 1 image per step (bounded CPU sample of the b128 batch)",
                   "model": args.model, "global_batch": 1, "parallelism": "cpu"},
        "efficiency": {"macs_per_image": macs, "gflops": 2 * macs * v / 1e9},
        "cpu_baseline": {"value": v, "unit": "images/s", "cores": threads, "kind": "port",
                         "sample": "1 image per step through the numpy oracle (oracle/model.py)"},
        "e2e": {"value": v, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- GPU arm


class ClockSampler:
    def __init__(self, device_index: int):
        self.idx = device_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 9:
                    continue
                sm.append(float(f[1]))
                mx = float(f[2])
                for nm, val in zip(names, f[5:9]):
                    if val.lower() == "active":
                        reasons.add(nm)
        except Exception:
            pass
        finally:
            try:
                os.unlink(self.path)
            except Exception:
                pass
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons)}


def run_gpu(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2404_03617_b200 import complexity
    from paper_2404_03617_b200.core import DeviceSpec, ExecutionScheme
    from paper_2404_03617_b200.scheduler import FusedNetwork

    B = args.batch
    net = _net(args.model)
    model = FusedNetwork(net, batch=B, seed=1234)
    gen = torch.Generator(device="cuda").manual_seed(rank)
    model.x.normal_(generator=gen)
    graph = model.capture()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        graph.replay()
    barrier()
    step_ms = []
    with ClockSampler(local) as clk:
        barrier()
        for _ in range(args.steps):
            flush.fill_(1)  # evict L2 between timed steps (outside the event pair)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            graph.replay()
            e1.record()
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
        barrier()
    clocks = clk.summary()
    ms = statistics.mean(step_ms)

    # ---- end to end through the public API: pinned host batches -> logits on
    # host (FusedNetwork.run_host_batches: every step's H2D copy and D2H read
    # are inside the timed region; step i+1's copy overlaps step i's forward)
    host_x = [torch.empty(model.x.shape, dtype=torch.float16, pin_memory=True) for _ in range(2)]
    for hx in host_x:
        hx.copy_(model.x.cpu())
    host_out = [torch.empty(model.output.shape, dtype=torch.float16, pin_memory=True) for _ in range(2)]
    model.run_host_batches([host_x[i % 2] for i in range(max(2, args.warmup))],
                           [host_out[i % 2] for i in range(max(2, args.warmup))])
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    model.run_host_batches([host_x[i % 2] for i in range(args.steps)], [host_out[i % 2] for i in range(args.steps)])
    e1.record()
    e1.synchronize()
    barrier()
    e2e = e0.elapsed_time(e1) / args.steps

    # ---- per-unit device times (dominant kernel roofline)
    unit_s = model.time_units(iters=10)

    if dist is not None:
        t = torch.tensor([ms, e2e], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e = float(t[0]), float(t[1])

    if rank == 0:
        peak_burst, peak_sust, hbm, peak_kind = _peaks()
        macs = complexity.network_macs(net)
        ops_batch = 2 * macs * B
        value = world * B / (ms / 1e3)
        dev = DeviceSpec("b200", peak_sust, hbm)
        wl = model.workloads(dev, ExecutionScheme.BLOCK_FUSION)
        # dominant kernel: identical units (same block, geometry) grouped, largest total share
        sig = lambda i: (repr(model.instances[i].block), model.instances[i].in_h, model.instances[i].in_w,
                         model.instances[i].in_channels, model.instances[i].out_channels)
        groups = {}
        for i in range(len(unit_s)):
            groups.setdefault(sig(i), []).append(i)
        members = max(groups.values(), key=lambda ix: sum(unit_s[i] for i in ix))
        di = members[len(members) // 2]
        dom = model.units[di]
        inst = model.instances[di]
        group_share = sum(unit_s[i] for i in members) / sum(unit_s)
        dom_ops = complexity.block_ops(inst.block, inst.dims(B), inst.out_channels)
        dom_bytes = wl[di].bytes
        intensity = dom_ops / dom_bytes
        bound = "tensor" if intensity >= dev.op_byte else "hbm"
        if bound == "tensor":
            achieved = dom_ops / unit_s[di] / 1e12
            peak = peak_burst / 1e12
            unit = "TFLOP/s"
        else:
            achieved = dom_bytes / unit_s[di] / 1e9
            peak = hbm / 1e9
            unit = "GB/s"
        traffic = None
        try:
            with open(os.path.join(HERE, "profiles", "ncu_traffic.json")) as fh:
                tkey = (f"{args.model}:{type(inst.block).__name__}:{inst.in_h}x{inst.in_w}x{inst.in_channels}"
                        f"->{inst.out_channels}")
                traffic = json.load(fh).get(tkey)
        except Exception:
            pass
        cpu = None
        if not args.skip_cpu:
            t_cpu, imgs, threads = cpu_sample(args.model, 1)
            cpu = {"value": imgs / t_cpu, "unit": "images/s", "cores": threads, "kind": "port",
                   "sample": f"{imgs} image through the numpy oracle of the same network (oracle/model.py), "
                             f"{t_cpu:.1f} s"}
        line = {
            "metric": f"images/sec ({args.model}@224 inference)",
            "value": value,
            "unit": "images/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "fp16",
            "data": "synthetic (N(0,1) images, fan-in scaled random-init weights)",
            "config": {
                "workload": f"{args.model}@224x224 forward, batch {B} per GPU, fp16 storage / fp32 accumulate",
                "model": args.model,
                "global_batch": B * world,
                "seq_len": None,
                "parallelism": f"dp{world} (independent image shards, no collective on the path)",
                "l2": "flushed between timed steps (256 MiB write outside the CUDA-event pair)",
            },
            "efficiency": {
                "macs_per_image": macs,
                "tflops": ops_batch / (ms / 1e3) / 1e12,
                "frac_of_datasheet_2250": ops_batch / (ms / 1e3) / PEAK_DATASHEET,
                f"frac_of_{peak_kind}_burst": ops_batch / (ms / 1e3) / peak_burst,
            },
            "roofline": {
                "kernel": f"{dom.label} ({type(inst.block).__name__} {inst.in_h}x{inst.in_w}x{inst.in_channels}"
                          f"->{inst.out_channels})",
                "bound": bound,
                "achieved": achieved,
                "peak": peak,
                "peak_kind": f"{peak_kind} {'bf16 burst' if bound == 'tensor' else 'HBM copy'}",
                "unit": unit,
                "frac": achieved / peak,
                "traffic": traffic,
                "algorithmic_flops_per_launch": dom_ops,
                "algorithmic_bytes_per_launch": dom_bytes,
                "share_of_step": group_share,
                "launches_in_group": len(members),
            },
            "e2e": {
                "value": world * B / (e2e / 1e3),
                "unit": "images/s",
                "h2d_bytes_per_step": int(model.x.numel() * 2),
                "d2h_bytes_per_step": int(model.output.numel() * 2),
            },
            "cpu_baseline": cpu,
            "clocks": clocks,
            "gpu_launches": model.launch_count() * args.steps,
            "units": {u.label: round(t * 1e6, 1) for u, t in zip(model.units, unit_s)},
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--model", default="convfirstnet-pico")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--skip-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
