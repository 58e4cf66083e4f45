"""``simulate`` on the B200: the reference's fusion-soundness check
(``cli.py:283-325`` ``cmd_simulate``) with both schedules executed on the
device — BLOCK_FUSION by the fused block kernels, LAYER_WISE by the
layer-by-layer device schedules (``WL_SCHEME_LAYER_WISE``) — plus each
schedule's tensor-machine DRAM plan and its measured device time.

    python -m paper_2404_03617_b200.simulate --block mbconv --channels 128 --size 14x14 --batch 128

Same arguments and exit codes as the reference subcommand (0 ok, 1 usage,
3 tolerance). The tolerance is the fp16 one of the parity tests (max-rel
1e-2; the reference's 1e-4 is its fp32/fp64 bound). There is no CPU path:
without a CUDA device the command exits with a usage error.
"""

from __future__ import annotations

import argparse
import sys

import numpy as np

from .core import FFN, ConvFirst, ExecutionScheme, MBConv, TensorDims
from . import machine

EXIT_OK, EXIT_USAGE, EXIT_TOLERANCE = 0, 1, 3
SIMULATE_TOLERANCE_FP16 = 1e-2


def _parse_size(text: str) -> tuple[int, int]:
    try:
        h, w = text.lower().split("x")
        return int(h), int(w)
    except ValueError:
        raise SystemExit(f"--size must look like 16x16, got {text!r}") from None


def build_block(args):
    if args.block == "ffn":
        return FFN(expansion=args.expansion, activation=args.activation or "relu")
    if args.block == "convfirst":
        return ConvFirst(group_width=args.group_width, expansion=args.expansion, activation=args.activation or "relu")
    if args.block == "mbconv":
        return MBConv(group_width=args.group_width, expansion=args.expansion, se_ratio=args.se_ratio,
                      activation=args.activation or "silu")
    raise SystemExit(f"unsupported block {args.block!r}")


def _device_ms(schedule, inputs, iters: int) -> float:
    """Mean device time of the schedule's launch (CUDA graph of one
    FusedBlock launch, inputs resident)."""
    import torch

    from .blocks import FusedBlock

    weights = {k: v for k, v in inputs.items() if k != "x"}
    m = FusedBlock(schedule.block, schedule.dims, out_channels=schedule.out_channels, weights=weights,
                   scheme=schedule.scheme)
    x = torch.from_numpy(np.ascontiguousarray(inputs["x"].reshape(m.in_shape))).half().cuda()
    out = torch.empty(m.out_shape, dtype=torch.float16, device="cuda")
    for _ in range(3):
        m.launch(x, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        m.launch(x, out)
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / iters


def main(argv=None) -> int:
    p = argparse.ArgumentParser(prog="simulate", description=__doc__.split("\n\n")[0])
    p.add_argument("--block", required=True, choices=("ffn", "convfirst", "mbconv"))
    p.add_argument("--channels", type=int, required=True)
    p.add_argument("--expansion", type=int, default=4)
    p.add_argument("--se-ratio", type=float, default=0.25)
    p.add_argument("--group-width", type=int, default=8)
    p.add_argument("--size", default="8x8", help="feature resolution HxW")
    p.add_argument("--batch", type=int, default=1)
    p.add_argument("--activation", default=None)
    p.add_argument("--scheme", choices=("layerwise", "blockfusion", "both"), default="both")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--backend", choices=("b200",), default="b200")
    p.add_argument("--time", type=int, default=0, help="also time each schedule over N device launches")
    args = p.parse_args(argv)

    import torch

    if not torch.cuda.is_available():
        print("simulate --backend b200 needs a CUDA device (there is no CPU path)", file=sys.stderr)
        return EXIT_USAGE
    h, w = _parse_size(args.size)
    dims = TensorDims(args.batch, h, w, args.channels)
    block = build_block(args)
    layerwise = machine.build_schedule(block, dims, ExecutionScheme.LAYER_WISE)
    fused = machine.build_schedule(block, dims, ExecutionScheme.BLOCK_FUSION)
    inputs = machine.random_inputs(layerwise, np.random.default_rng(args.seed))
    out_lw = machine.execute_numeric(layerwise, inputs)
    out_bf = machine.execute_numeric(fused, inputs)
    denom = max(float(np.abs(out_lw).max()), 1e-12)
    rel_err = float(np.abs(out_lw - out_bf).max()) / denom
    for name, schedule in (("layerwise", layerwise), ("blockfusion", fused)):
        if args.scheme not in ("both", name):
            continue
        report = machine.simulate_traffic(schedule)
        line = (f"{name:12s} dram {report.dram_bytes} B  global<->local {report.global_local_bytes} B  "
                f"macs {report.mac_ops}  syncs {report.sync_count}")
        if args.time and block.__class__ is not FFN:
            line += f"  device {_device_ms(schedule, inputs, args.time) * 1e3:.1f} us"
        print(line)
    print(f"fused vs layer-wise max relative error (device, fp16): {rel_err:.3e} (seed {args.seed})")
    if not np.isfinite(rel_err) or rel_err > SIMULATE_TOLERANCE_FP16:
        print(f"FAIL: exceeds tolerance {SIMULATE_TOLERANCE_FP16:g}", file=sys.stderr)
        return EXIT_TOLERANCE
    return EXIT_OK


if __name__ == "__main__":
    sys.exit(main())
