"""simulate_traffic / dram_bytes_by_role of the UNMODIFIED reference
(machine.py:826-897) on a grid of blocks, shapes, schemes and partitions ->
tests/golden/traffic.json. Run in the build container:
    python tests/golden/make_traffic_golden.py
"""

import itertools
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    from waterline.core import ConvFirst, ExecutionScheme, FFN, MBConv, TensorDims
    from waterline.machine import build_schedule, dram_bytes_by_role, simulate_traffic

    blocks = [("FFN", dict(expansion=4, activation="relu")), ("FFN", dict(expansion=3, activation="silu")),
              ("ConvFirst", dict(group_width=8, expansion=6, stride=1)), ("ConvFirst", dict(group_width=1, expansion=4)),
              ("ConvFirst", dict(group_width=8, expansion=3, stride=2)),
              ("MBConv", dict(group_width=8, expansion=4, se_ratio=0.25)),
              ("MBConv", dict(group_width=1, expansion=6, se_ratio=0.25)),
              ("MBConv", dict(group_width=8, expansion=4, se_ratio=0.25, stride=2))]
    kinds = {"FFN": FFN, "ConvFirst": ConvFirst, "MBConv": MBConv}
    dims = [(2, 8, 8, 32), (1, 14, 14, 64), (3, 6, 10, 16)]
    out = []
    for (kind, params), d, scheme in itertools.product(blocks, dims, ExecutionScheme):
        block = kinds[kind](**params)
        td = TensorDims(*d)
        k = 2 * d[3] if params.get("stride") == 2 else None
        procs = [None]
        if scheme == ExecutionScheme.BLOCK_FUSION and kind == "ConvFirst" and params.get("stride", 1) == 1:
            procs += [2, 4]
        if scheme == ExecutionScheme.BLOCK_FUSION and kind == "MBConv":
            procs += [1, 2]
        for p in procs:
            try:
                s = build_schedule(block, td, scheme, out_channels=k, processors=p)
            except ValueError:
                continue
            t = simulate_traffic(s)
            out.append({"block": kind, "params": params, "dims": list(d), "scheme": scheme.value,
                        "out_channels": k, "processors": p,
                        "traffic": [t.dram_global_bytes, t.global_local_bytes, t.mac_ops, t.sync_count],
                        "by_role": dram_bytes_by_role(s)})
    with open(os.path.join(HERE, "traffic.json"), "w") as fh:
        json.dump(out, fh, indent=0)
    print(len(out), "cases")


if __name__ == "__main__":
    main()
