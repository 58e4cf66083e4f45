"""The accounting drop-ins (simulate_traffic, dram_bytes_by_role,
validate_schedule; machine.py:786-897) against the UNMODIFIED reference on
a grid of blocks / shapes / schemes / partitions (tests/golden/traffic.json,
made by tests/golden/make_traffic_golden.py), and the FFN helpers against
the SPEC known answers."""

import json
import os

import numpy as np
import pytest

from paper_2404_03617_b200.core import ConvFirst, ExecutionScheme, FFN, MBConv, TensorDims
from paper_2404_03617_b200.machine import (
    ScheduleError, build_schedule, dram_bytes_by_role, ffn_fused, ffn_layerwise, simulate_traffic,
    validate_schedule,
)

with open(os.path.join(os.path.dirname(__file__), "golden", "traffic.json")) as fh:
    CASES = json.load(fh)
KINDS = {"FFN": FFN, "ConvFirst": ConvFirst, "MBConv": MBConv}


@pytest.mark.parametrize("case", CASES, ids=[f"{c['block']}-{c['scheme']}-{c['dims']}-{c['processors']}-{i}"
                                              for i, c in enumerate(CASES)])
def test_traffic_matches_reference(case):
    s = build_schedule(KINDS[case["block"]](**case["params"]), TensorDims(*case["dims"]),
                       ExecutionScheme(case["scheme"]), out_channels=case["out_channels"],
                       processors=case["processors"])
    t = simulate_traffic(s)
    assert [t.dram_global_bytes, t.global_local_bytes, t.mac_ops, t.sync_count] == case["traffic"]
    assert t.dram_bytes == case["traffic"][0]
    assert dram_bytes_by_role(s) == case["by_role"]


def test_validate_schedule_rejects_a_broken_table():
    s = build_schedule(ConvFirst(8, 6), TensorDims(1, 8, 8, 16))
    validate_schedule(s)
    from dataclasses import replace

    with pytest.raises(ScheduleError, match="undeclared"):
        validate_schedule(replace(s, tensors=tuple(t for t in s.tensors if t.name != "u")))


def test_ffn_known_answers():
    one = np.array([[1.0]])
    assert ffn_layerwise(one, np.array([[2.0]]), np.array([[3.0]]), np.array([1.0]), np.array([-1.0])).tolist() == [[8.0]]
    rng = np.random.default_rng(0)
    x, u, v = rng.standard_normal((6, 4)), rng.standard_normal((4, 12)), rng.standard_normal((12, 4))
    a, b = rng.standard_normal(12), rng.standard_normal(4)
    lw = ffn_layerwise(x, u, v, a, b)
    assert np.array_equal(ffn_fused(x, u, v, a, b, chunk=12), lw)  # chunk == hidden is bit-identical
    assert np.abs(ffn_fused(x, u, v, a, b, chunk=1) - lw).max() <= 1e-5 * np.abs(lw).max()
    with pytest.raises(ValueError):
        ffn_fused(x, u, v, a, b, chunk=0)
    with pytest.raises(ValueError):
        ffn_layerwise(x, u[:3], v, a, b)
