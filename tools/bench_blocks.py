"""BASELINE configs 1 and 2 as single-block measurements on one B200:
C1 ConvNeXt-style block 56x56x96 (dw7x7 -> LN -> 1x1 4x -> GELU -> 1x1 + res), batch 8;
C2 MBConv 28x28x80 (group width 1 = depthwise, SE 0.25), batch 128.
Per config: a stage of 8 copies with distinct weights (so weights are not L2-hot,
SURVEY 8d), device-timed with CUDA events over graph replays, L2 flushed between
timed replays; algorithmic FLOPs / bytes from complexity.block_costs."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_03617_b200 import complexity  # noqa: E402
from paper_2404_03617_b200.blocks import FusedBlock  # noqa: E402
from paper_2404_03617_b200.core import ConvNeXtBlock, DeviceSpec, ExecutionScheme, MBConv, TensorDims  # noqa: E402

peaks = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")) else {}
CONFIGS = {
    "C1 convnext 56x56x96 b8": (ConvNeXtBlock(7, 4, "gelu"), TensorDims(8, 56, 56, 96)),
    "C2 mbconv T=1 28x28x80 b128": (MBConv(1, 4, 0.25), TensorDims(128, 28, 28, 80)),
    "C2' mbconv T=8 28x28x80 b128": (MBConv(8, 4, 0.25), TensorDims(128, 28, 28, 80)),
}
dev = DeviceSpec("acct", 1.0, 1.0, bytes_per_element=2)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, (blk, dims) in CONFIGS.items():
    mods = [FusedBlock(blk, dims, seed=s) for s in range(8)]
    xs = [torch.randn(*m.in_shape, device="cuda").half() for m in mods[:1]]
    bufs = [xs[0]] + [torch.empty(m.out_shape, dtype=torch.float16, device="cuda") for m in mods]
    ws = max(m.workspace.numel() for m in mods)
    wsb = torch.zeros(ws, dtype=torch.uint8, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3):
            for i, m in enumerate(mods):
                m.launch(bufs[i], bufs[i + 1], wsb)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i, m in enumerate(mods):
                m.launch(bufs[i], bufs[i + 1], wsb)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3 / len(mods))
    t = sorted(ts)[len(ts) // 2]
    cost = complexity.block_costs(blk, dims, ExecutionScheme.BLOCK_FUSION, dev)
    flops = cost.ops if hasattr(cost, "ops") else 2 * cost.macs
    print(json.dumps({"config": name, "us_per_block": round(t * 1e6, 2), "images_per_s": round(dims.n / t),
                      "tflops": round(flops / t / 1e12, 1), "hbm_gbs": round(cost.bytes / t / 1e9, 1),
                      "algorithmic_flops": flops, "algorithmic_bytes": cost.bytes}), flush=True)
