"""ConvNeXt-T (BASELINE config 4) on the CPU: the unit plan, the MAC count the
efficiency numerator uses, tensor tables, C-ABI descriptors, and the
layer-scale fold (exact through the oracle)."""

import numpy as np
import pytest

import oracle
from oracle import model as om
from paper_2404_03617_b200.convnext import ConvNeXtSpec, convnext_tiny, fold_layer_scale, network_macs
from paper_2404_03617_b200.core import ConvNeXtBlock, Downsample, LNHead, PatchifyStem, TensorDims
from paper_2404_03617_b200.machine import block_descriptor, build_schedule, device_binding


def test_convnext_tiny_plan():
    units = convnext_tiny(224).plan()
    labels = [u.label for u in units]
    assert labels[0] == "stem" and labels[-1] == "head"
    assert sum(isinstance(u.block, ConvNeXtBlock) for u in units) == 18
    assert [u.label for u in units if isinstance(u.block, Downsample)] == ["ds1", "ds2", "ds3"]
    widths = {(u.in_h, u.in_channels) for u in units if isinstance(u.block, ConvNeXtBlock)}
    assert widths == {(56, 96), (28, 192), (14, 384), (7, 768)}
    # consecutive units chain: out of one = in of the next
    for a, b in zip(units, units[1:]):
        assert (a.out_h, a.out_w, a.out_channels) == (b.in_h, b.in_w, b.in_channels)


def test_convnext_tiny_macs():
    # 4.456 GMAC/img at 224 (timm / fvcore count convs + linears)
    assert network_macs(convnext_tiny(224)) == 4_455_531_264
    assert abs(network_macs(convnext_tiny(288)) / network_macs(convnext_tiny(224)) - (288 / 224) ** 2) < 2e-3


def test_spec_validation():
    with pytest.raises(ValueError):
        ConvNeXtSpec("bad", (100, 100))
    with pytest.raises(ValueError):
        ConvNeXtSpec("bad", (224, 224), depths=(1, 1), dims=(8,))


@pytest.mark.parametrize("block,dims,k,out", [
    (PatchifyStem(96), TensorDims(2, 224, 224, 3), None, (2, 56, 56, 96)),
    (Downsample(192), TensorDims(2, 56, 56, 96), None, (2, 28, 28, 192)),
    (LNHead(1000), TensorDims(2, 7, 7, 768), None, (2, 1000)),
    (ConvNeXtBlock(7, 4, "gelu"), TensorDims(2, 14, 14, 384), None, (2, 14, 14, 384)),
])
def test_schedules_and_descriptors(block, dims, k, out):
    pytest.importorskip("ctypes")
    s = build_schedule(block, dims, out_channels=k)
    assert s.out_dims == out
    b = device_binding(s)
    assert not b.padded
    d = block_descriptor(block, dims, s.out_channels)
    assert d.n == dims.n and d.c == dims.c


def test_layer_scale_fold_is_exact():
    rng = np.random.default_rng(0)
    c = 16
    x = rng.standard_normal((1, 6, 6, c)).astype(np.float32)
    w = {"w_conv": rng.standard_normal((c, 7, 7, 1)).astype(np.float32) / 7, "b_conv": rng.standard_normal(c),
         "ln_gamma": np.ones(c), "ln_beta": np.zeros(c), "u": rng.standard_normal((c, 4 * c)) / 4,
         "a": rng.standard_normal(4 * c), "v": rng.standard_normal((4 * c, c)) / 8, "b": rng.standard_normal(c)}
    gamma = rng.uniform(0.5, 1.5, c)
    blk = ConvNeXtBlock(7, 4, "gelu")
    folded = om.unit_forward(blk, fold_layer_scale(w, gamma), x)
    plain = om.unit_forward(blk, w, x) - x
    np.testing.assert_allclose(folded - x, plain * gamma, rtol=1e-4, atol=1e-5)


def test_network_oracle_runs_small():
    spec = ConvNeXtSpec("mini", (64, 64), depths=(1, 1, 1, 1), dims=(16, 32, 64, 128), num_classes=24)
    from paper_2404_03617_b200.blocks import init_weights

    rng = np.random.default_rng(3)
    units = spec.plan()
    wts = {u.label: init_weights(build_schedule(u.block, u.dims(1), out_channels=u.out_channels), rng) for u in units}
    out = om.network_forward(units, wts, rng.standard_normal((1, 64, 64, 3)).astype(np.float32))
    assert out.shape == (1, 24) and np.isfinite(out).all()
