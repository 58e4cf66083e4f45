"""Domain model + cost model: drop-in parity with the reference (golden
values from tests/golden/make_cost_golden.py) and the reference tests'
known answers (tests/test_complexity.py, test_core.py, test_perf.py)."""

from dataclasses import replace

import pytest

from oracle.fixtures import load_costs
from paper_2404_03617_b200 import complexity as cx, perf, zoo
from paper_2404_03617_b200.core import (
    ConvFirst, ConvNeXtBlock, ConvSpec, DeviceSpec, ExecutionScheme, FFN, Head, MBConv, NetworkSpec,
    NetworkValidationError, StageSpec, Stem, TensorDims, expand_network, network_from_json, network_to_json,
    plan_blocks, validate_network, device_from_json, device_to_json,
)

COSTS = load_costs()
DEV = DeviceSpec("b200-datasheet", 2.25e15, 8.0e12)


@pytest.mark.parametrize("key", sorted(COSTS))
def test_cost_model_matches_reference(key):
    name, res = key.split("@")
    net = replace(zoo.from_name(name), input_resolution=(int(res), int(res)))
    ref = COSTS[key]
    assert cx.network_macs(net) == ref["macs"]
    assert cx.count_params(net) == ref["params"]
    for sch in ExecutionScheme:
        wl = expand_network(net, 128, sch, DEV)
        assert [[w.label, w.ops, w.bytes] for w in wl] == ref[sch.value]["workloads"]
        v = perf.waterline(wl, DEV)
        assert v.max_efficiency == pytest.approx(ref[sch.value]["max_efficiency"], rel=1e-12)
        assert v.mediant_intensity == pytest.approx(ref[sch.value]["mediant"], rel=1e-12)


def test_reference_known_answers():
    assert cx.conv_ops(ConvSpec(3, 16, 3, 3, None, stride=2), TensorDims(1, 256, 256, 3)) == 14_155_776
    assert cx.conv_ops(ConvSpec(16, 16, 3, 3, group_width=8), TensorDims(1, 128, 128, 16)) == 37_748_736
    assert cx.conv_ops(ConvSpec(1, 1, 1, 1, None, has_bias=True), TensorDims(1, 1, 1, 1)) == 3
    by = {c.label: c.ops for c in cx.block_costs(MBConv(8, 4, 0.25, 1), TensorDims(1, 16, 16, 128),
                                                 ExecutionScheme.LAYER_WISE, DEV)}
    assert by["se"] == 4 * 512 * 32
    assert by["exp"] == pytest.approx(33.55e6, rel=0.005)
    assert cx.network_macs(zoo.build(zoo.ZooId.CONVFIRSTNET_PICO)) == pytest.approx(0.86e9, rel=0.02)
    net = NetworkSpec("stem-only", (256, 256), Stem(16), (), None)
    assert cx.network_macs(net) == pytest.approx(7.08e6, rel=0.005)


def test_pico_at_224_has_30_units_and_the_expected_geometry():
    units = plan_blocks(zoo.at_resolution(zoo.from_name("convfirstnet-pico"), 224))
    assert len(units) == 30
    assert [u.label for u in units[:3]] == ["stem", "s1b0", "s2b0"]
    s4 = [u for u in units if u.label.startswith("s4")]
    assert (s4[0].in_h, s4[0].stride, s4[1].in_h) == (28, 2, 14)
    assert units[-1].label == "head" and units[-1].in_h == 7


def test_stemless_network_binds_stage_channels():
    # the reference's own expectation (tests/test_core.py:149-152)
    net = zoo.build_stack(ConvFirst(8, 6), 8, TensorDims(128, 64, 64, 32))
    assert plan_blocks(net)[0].in_channels == 32
    one = NetworkSpec("one", (8, 8), None, (StageSpec(FFN(4), 1, 16),), None)
    for sch in ExecutionScheme:
        assert len(expand_network(one, 1, sch, DEV)) == (2 if sch == ExecutionScheme.LAYER_WISE else 1)


def test_validation_errors_are_structured():
    bad = NetworkSpec("bad", (30, 30), Stem(16), (StageSpec(ConvFirst(5, 6), 1, 16),), Head())
    v = validate_network(bad)
    assert any("group width 5" in s for s in v)
    with pytest.raises(NetworkValidationError) as e:
        plan_blocks(bad)
    assert e.value.violations == v
    with pytest.raises(ValueError):
        TensorDims(0, 1, 1, 1)
    with pytest.raises(ValueError):
        DeviceSpec("x", 0, 1)


def test_json_round_trips():
    for z in zoo.ZooId:
        net = zoo.build(z)
        assert network_from_json(network_to_json(net)) == net
    cn = NetworkSpec("cnx", (56, 56), None, (StageSpec(ConvNeXtBlock(), 3, 96),), None)
    assert network_from_json(network_to_json(cn)) == cn
    assert device_from_json(device_to_json(DEV)) == DEV


def test_convnext_block_costs_fused_bytes_and_ops():
    dims = TensorDims(8, 56, 56, 96)
    fused = cx.block_costs(ConvNeXtBlock(), dims, ExecutionScheme.BLOCK_FUSION, DEV)
    lw = cx.block_costs(ConvNeXtBlock(), dims, ExecutionScheme.LAYER_WISE, DEV)
    assert fused.ops == sum(c.ops for c in lw)
    assert fused.bytes < sum(c.bytes for c in lw)
    # dw7x7 + 2 x (96 x 384) per pixel ~ 3.9 GFLOP at b8
    assert fused.ops == pytest.approx(3.935e9, rel=0.01)


def test_waterline_properties(b200):
    wl = expand_network(zoo.at_resolution(zoo.from_name("convfirstnet-pico"), 224), 128,
                        ExecutionScheme.BLOCK_FUSION, b200)
    v = perf.waterline(wl, b200)
    assert 0 < v.max_efficiency <= perf.roofline_efficiency(wl, b200) <= 1
    pts = perf.opbyte_sweep(wl, b200, 10, 1000, 5)
    assert all(p.waterline_efficiency <= p.roofline_efficiency + 1e-12 for p in pts)
    mk = perf.measured_waterline(wl, [2 * x.attainable_latency for x in v.verdicts], b200)
    assert all(m.efficiency == pytest.approx(0.5) for m in mk)
