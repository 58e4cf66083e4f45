"""Cost-model golden values from the UNMODIFIED reference (run in the build
container): network MACs / params, expand_network workloads under both
schemes and the waterline verdicts for every zoo model at 224 and 256, on
the B200 datasheet device. Written to tests/golden/costs.json."""

from __future__ import annotations

import json
import os
import sys
from dataclasses import replace

sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    from waterline import complexity as cx, perf, zoo
    from waterline.core import DeviceSpec, ExecutionScheme, expand_network

    dev = DeviceSpec("b200-datasheet", 2.25e15, 8.0e12)
    out = {}
    for z in zoo.ZooId:
        for res in (224, 256):
            net = replace(zoo.build(z), input_resolution=(res, res))
            key = f"{z.value}@{res}"
            entry = {"macs": cx.network_macs(net), "params": cx.count_params(net)}
            for sch in ExecutionScheme:
                wl = expand_network(net, 128, sch, dev)
                v = perf.waterline(wl, dev)
                entry[sch.value] = {
                    "workloads": [[w.label, w.ops, w.bytes] for w in wl],
                    "max_efficiency": v.max_efficiency,
                    "total_latency": v.total_latency,
                    "mediant": v.mediant_intensity,
                }
            out[key] = entry
    with open(os.path.join(HERE, "costs.json"), "w") as fh:
        json.dump(out, fh)
    print("wrote", len(out), "models")


if __name__ == "__main__":
    main()
