"""Generate golden vectors from the UNMODIFIED reference implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

For every case, inputs come from the reference's own ``random_inputs``
(machine.py:1064-1070) on the LAYER_WISE schedule, are rounded to fp16 (so
the GPU path consumes exactly the same values), and the reference's
``execute_numeric`` (machine.py:1053) evaluates both the LAYER_WISE and the
BLOCK_FUSION schedules. The .npz files are committed; the GPU box never reads
/root/reference.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    sys.path.insert(0, REF)
    from waterline.core import ConvFirst, ExecutionScheme, FFN, MBConv, TensorDims  # noqa: E402
    from waterline.machine import build_schedule, execute_numeric, random_inputs, simulate_traffic  # noqa: E402

    cases = [
        ("convfirst_t8_a6_relu", ConvFirst(8, 6, 1, "relu"), (2, 8, 8, 16), 0),
        ("convfirst_t8_a3_relu_rect", ConvFirst(8, 3, 1, "relu"), (1, 12, 10, 32), 1),
        ("convfirst_t1_a4_relu", ConvFirst(1, 4, 1, "relu"), (2, 8, 8, 16), 2),
        ("convfirst_t8_a4_silu_7x7", ConvFirst(8, 4, 1, "silu"), (2, 7, 7, 24), 3),
        ("convfirst_t8_a6_relu_c48", ConvFirst(8, 6, 1, "relu"), (1, 14, 14, 48), 4),
        ("mbconv_t8_a4_se25", MBConv(8, 4, 0.25, 1, "silu"), (2, 7, 7, 32), 5),
        ("mbconv_t1_a4_se25", MBConv(1, 4, 0.25, 1, "silu"), (2, 8, 8, 16), 6),
        ("mbconv_t8_a4_se25_14", MBConv(8, 4, 0.25, 1, "silu"), (1, 14, 14, 48), 7),
        ("mbconv_t8_a4_se25_c128_7", MBConv(8, 4, 0.25, 1, "silu"), (2, 7, 7, 128), 8),
        ("ffn_a4_relu", FFN(4, "relu"), (1, 8, 8, 16), 9),
        # processors > 1: the channel-partitioned ConvFirst scaling schedule
        # (machine.py:528-569) and the explicitly partitioned MBConv (machine.py:649-660)
        ("convfirst_t8_a6_relu_scaling_p2", ConvFirst(8, 6, 1, "relu"), (1, 8, 8, 32), 10, 2),
        ("convfirst_t8_a4_relu_scaling_p4", ConvFirst(8, 4, 1, "relu"), (2, 6, 6, 64), 11, 4),
        ("mbconv_t8_a4_se25_p2", MBConv(8, 4, 0.25, 1, "silu"), (2, 7, 7, 32), 12, 2),
    ]
    index = {}
    for case in cases:
        name, block, dims, seed = case[:4]
        procs = case[4] if len(case) > 4 else None
        td = TensorDims(*dims)
        lw = build_schedule(block, td, ExecutionScheme.LAYER_WISE)
        bf = build_schedule(block, td, ExecutionScheme.BLOCK_FUSION)
        inputs = random_inputs(lw, np.random.default_rng(seed))
        inputs = {k: v.astype(np.float16).astype(np.float32) for k, v in inputs.items()}
        out_lw = execute_numeric(lw, inputs)
        if procs:  # the partitioned schedule is the one evaluated as "fused"
            out_bf = execute_numeric(build_schedule(block, td, ExecutionScheme.BLOCK_FUSION, processors=procs), inputs)
        else:
            out_bf = execute_numeric(bf, inputs)
        traffic = simulate_traffic(bf)
        meta = {
            "block": type(block).__name__,
            "params": {k: getattr(block, k) for k in block.__dataclass_fields__},
            "dims": list(dims),
            "seed": seed,
            "fused_dram_bytes": traffic.dram_bytes,
            "macs": traffic.mac_ops,
            "fused_vs_layerwise_max_abs": float(np.max(np.abs(out_lw - out_bf))),
        }
        if procs:
            meta["processors"] = procs
        np.savez_compressed(
            os.path.join(HERE, f"{name}.npz"),
            out_layerwise=out_lw,
            out_fused=out_bf,
            meta=json.dumps(meta),
            **{"in_" + k: v.astype(np.float16) for k, v in inputs.items()},
        )
        index[name] = meta
        print(name, dims, "max|out|=%.3g" % np.abs(out_lw).max(), "lw-vs-fused %.2g" % meta["fused_vs_layerwise_max_abs"])
    with open(os.path.join(HERE, "index.json"), "w") as fh:
        json.dump(index, fh, indent=1, sort_keys=True)
    make_big(build_schedule, execute_numeric, random_inputs, ConvFirst, MBConv, TensorDims, ExecutionScheme)


# BASELINE.json configs at full size: the whole batch's inputs come from the
# reference's own random_inputs stream (seeded; our machine.random_inputs is
# bit-identical, tests/test_machine_api.py), the unmodified reference
# execute_numeric (LAYER_WISE) runs on the picked images only (images are
# independent), and only those outputs are stored. The GPU test regenerates
# the full batch from the seed, runs it at full batch and compares the picks.
BIG_CASES = [
    # config 1's closest reference form (3x3 depthwise ConvFirst, no LN) and the ConvFirstNet form
    ("big_convfirst_t1_a4_56x56x96_b8", "ConvFirst", dict(group_width=1, expansion=4, stride=1, activation="relu"),
     (8, 56, 56, 96), 21, [0, 7]),
    ("big_convfirst_t8_a6_56x56x96_b8", "ConvFirst", dict(group_width=8, expansion=6, stride=1, activation="relu"),
     (8, 56, 56, 96), 22, [0, 7]),
    # config 2: MBConv(1, 4, .25) 28x28x80 at batch 128
    ("big_mbconv_t1_a4_28x28x80_b128", "MBConv", dict(group_width=1, expansion=4, se_ratio=0.25, stride=1,
                                                       activation="silu"), (128, 28, 28, 80), 23, [0, 63, 127]),
    # the ConvFirstNet-Pico 14x14 MBConv at batch 128
    ("big_mbconv_t8_a4_14x14x128_b128", "MBConv", dict(group_width=8, expansion=4, se_ratio=0.25, stride=1,
                                                        activation="silu"), (128, 14, 14, 128), 24, [0, 63, 127]),
]


def make_big(build_schedule, execute_numeric, random_inputs, ConvFirst, MBConv, TensorDims, ExecutionScheme):
    kinds = {"ConvFirst": ConvFirst, "MBConv": MBConv}
    for name, kind, params, dims, seed, picks in BIG_CASES:
        block = kinds[kind](**params)
        lw = build_schedule(block, TensorDims(*dims), ExecutionScheme.LAYER_WISE)
        ins = random_inputs(lw, np.random.default_rng(seed))
        ins = {k: v.astype(np.float16).astype(np.float32) for k, v in ins.items()}
        sub = dict(ins, x=ins["x"][picks])
        lw_sub = build_schedule(block, TensorDims(len(picks), *dims[1:]), ExecutionScheme.LAYER_WISE)
        out = execute_numeric(lw_sub, sub)
        meta = {"block": kind, "params": params, "dims": list(dims), "seed": seed, "picks": picks,
                "x_checksum": float(ins["x"].astype(np.float64).sum()),
                "w_checksum": float(sum(v.astype(np.float64).sum() for k, v in ins.items() if k != "x"))}
        np.savez_compressed(os.path.join(HERE, "big", f"{name}.npz"), out_picked=out, meta=json.dumps(meta))
        print(name, dims, picks, "max|out|=%.3g" % np.abs(out).max())


if __name__ == "__main__":
    main()
