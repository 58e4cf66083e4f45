"""Zero channel padding (machine.device_binding): ConvFirstNet-Nano/Tiny's
C % 16 != 0 widths run on the device as the next multiple of 16. Checked on
the CPU through the oracle: the padded block's real channels equal the
unpadded block, its padded channels are exactly zero, and every padded
descriptor is accepted by the library's launch planner."""

import ctypes

import numpy as np
import pytest

from oracle import model as om
from paper_2404_03617_b200 import _lib, zoo
from paper_2404_03617_b200.blocks import init_weights
from paper_2404_03617_b200.core import ConvFirst, ConvNeXtBlock, Head, MBConv, Stem, TensorDims, plan_blocks
from paper_2404_03617_b200.machine import ScheduleError, build_schedule, device_binding, device_channels, weight_names

CASES = [
    (Stem(24), TensorDims(1, 16, 16, 3), None),
    (ConvFirst(8, 3), TensorDims(1, 12, 10, 24), None),
    (ConvFirst(8, 6, 2), TensorDims(1, 12, 12, 24), 48),
    (ConvFirst(8, 6, 2), TensorDims(1, 12, 12, 48), 72),
    (ConvFirst(8, 6), TensorDims(1, 7, 7, 72), None),
    (MBConv(8, 4, 0.25, 2), TensorDims(1, 8, 8, 72), 192),
    (MBConv(8, 4, 0.25), TensorDims(1, 7, 7, 24), None),
    (Head(64, 10), TensorDims(2, 3, 3, 72), None),
]


def test_device_channels():
    assert [device_channels(c) for c in (16, 24, 48, 72, 160, 192, 8)] == [16, 32, 48, 80, 160, 192, 16]


@pytest.mark.parametrize("block,dims,k", CASES, ids=[f"{type(c[0]).__name__}-{c[1].c}-{c[2]}" for c in CASES])
def test_padded_block_equals_real_block(block, dims, k):
    rng = np.random.default_rng(0)
    s = build_schedule(block, dims, out_channels=k)
    w = init_weights(s, rng)
    x = rng.standard_normal((dims.n, dims.h, dims.w, dims.c)).astype(np.float32)
    b = device_binding(s)
    assert b.padded
    dw = dict(zip(weight_names(s), b.device_weights(w)))
    real = om.unit_forward(block, w, x)
    padded = om.unit_forward(b.block, dw, b.device_input(x))
    if padded.ndim == 4:
        assert padded.shape[3] == b.k
        assert not padded[..., real.shape[3]:].any()
    np.testing.assert_allclose(b.real_output(padded), real, rtol=1e-5, atol=1e-5)


def test_layernorm_blocks_refuse_padding():
    with pytest.raises(ScheduleError):
        device_binding(build_schedule(ConvNeXtBlock(7, 4, "gelu"), TensorDims(1, 8, 8, 24)))


@pytest.mark.parametrize("res", [224, 256])
@pytest.mark.parametrize("model", ["convfirstnet-pico", "convfirstnet-nano", "convfirstnet-tiny", "convfirstnet-small"])
def test_zoo_models_plan_at_b128(model, res):
    """Every unit of every zoo model has a launch plan at the BASELINE batch,
    at 224 and at the reference's native 256 (zoo.py:10)."""
    L = _lib.lib()
    net = zoo.at_resolution(zoo.from_name(model), res)
    for inst in plan_blocks(net):
        b = device_binding(build_schedule(inst.block, inst.dims(128), out_channels=inst.out_channels))
        assert L.wl_validate(ctypes.byref(b.desc)) == 0, (inst.label, _lib.last_error())


@pytest.mark.parametrize("model", ["convfirstnet-pico", "convfirstnet-small"])
def test_zoo_launch_plan_is_one_kernel_per_block(model):
    """The model-level scheduler's promise (one fused launch per block, two
    for the head) holds for the plans the library picks at b128."""
    L = _lib.lib()
    net = zoo.at_resolution(zoo.from_name(model), 224)
    counts = {}
    for inst in plan_blocks(net):
        b = device_binding(build_schedule(inst.block, inst.dims(128), out_channels=inst.out_channels))
        counts[inst.label] = L.wl_kernel_launches(ctypes.byref(b.desc))
    assert counts.pop("head") == 2
    assert set(counts.values()) == {1}, counts
