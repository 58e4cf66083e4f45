"""The C ABI (include/wlfuse.h) without a GPU: the library loads, exports
every declared symbol, validates descriptors with the reference's error
mapping, and packs weights deterministically."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2404_03617_b200 import _lib
from paper_2404_03617_b200.core import ConvFirst, ExecutionScheme, Head, MBConv, Stem, TensorDims
from paper_2404_03617_b200.machine import ScheduleError, block_descriptor, build_schedule, random_inputs, weight_names

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "wlfuse.h")


def declared_symbols():
    return sorted(set(re.findall(r"WL_API\s+[\w\s\*]+?\b(wl_\w+)\s*\(", open(HEADER).read())))


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 15
    so = ctypes.CDLL(_lib.LIB_PATH)
    for s in syms:
        assert hasattr(so, s), s
    assert sorted(_lib.EXPORTS) == syms
    assert _lib.lib().wl_version() == 1


def _desc(block, dims, k=None):
    return block_descriptor(block, dims, k if k is not None else dims.c)


def test_validate_maps_errors_like_the_reference():
    L = _lib.lib()
    d = _desc(ConvFirst(8, 6), TensorDims(1, 16, 16, 32))
    assert L.wl_validate(ctypes.byref(d)) == 0
    d.c = 36  # group width 8 does not divide 36 -> ValueError in the reference
    with pytest.raises(ValueError):
        _lib.check(L.wl_validate(ctypes.byref(d)))
    d = _desc(ConvFirst(8, 6), TensorDims(1, 16, 16, 32))
    d.group_width = 4  # valid block, no kernel -> ScheduleError (not executable)
    with pytest.raises(ScheduleError):
        _lib.check(L.wl_validate(ctypes.byref(d)))
    d = _desc(ConvFirst(8, 6), TensorDims(1, 16, 16, 32))
    d.k = 64  # stride-1 blocks keep their channel count
    with pytest.raises(ValueError):
        _lib.check(L.wl_validate(ctypes.byref(d)))
    d.kind = 99
    with pytest.raises(ValueError):
        _lib.check(L.wl_validate(ctypes.byref(d)))


@pytest.mark.parametrize(
    "block,dims,k",
    [
        (ConvFirst(8, 6), TensorDims(2, 56, 56, 32), None),
        (ConvFirst(8, 6, 2), TensorDims(2, 112, 112, 16), 32),
        (MBConv(8, 4, 0.25), TensorDims(128, 14, 14, 128), None),
        (MBConv(8, 4, 0.25, 2), TensorDims(128, 28, 28, 48), 128),
        (MBConv(1, 4, 0.25), TensorDims(128, 28, 28, 80), None),
        (Stem(16), TensorDims(128, 224, 224, 3), 16),
        (Head(), TensorDims(128, 7, 7, 128), 1000),
    ],
)
def test_pack_is_deterministic_and_sized(block, dims, k):
    s = build_schedule(block, dims, out_channels=k)
    d = block_descriptor(block, dims, s.out_channels)
    ins = random_inputs(s, np.random.default_rng(0))
    w = [ins[n] for n in weight_names(s)]
    a = _lib.pack_weights(d, w)
    b = _lib.pack_weights(d, w)
    assert a.nbytes == _lib.lib().wl_packed_bytes(ctypes.byref(d)) and np.array_equal(a, b)
    assert a.any()
    with pytest.raises(ValueError):
        _lib.pack_weights(d, w[:-1])
    n, h, ww, c = _lib.output_dims(d)
    assert (n, h, ww, c)[0] == dims.n


def test_output_dims_and_workspace():
    L = _lib.lib()
    d = _desc(MBConv(8, 4, 0.25, 2), TensorDims(4, 28, 28, 48), 128)
    assert _lib.output_dims(d) == (4, 14, 14, 128)
    ws = L.wl_workspace_bytes(ctypes.byref(d))
    assert ws >= 4 * 14 * 14 * 192 * 2 + 4 * 192 * 4  # L2-resident hidden + SE pool
    d = _desc(ConvFirst(8, 6), TensorDims(4, 28, 28, 48))
    assert L.wl_workspace_bytes(ctypes.byref(d)) == 0  # fully fused


def test_kernel_launches_per_block():
    """wl_kernel_launches reports the planned launches (host-side, no GPU):
    one per fused block, two for the head (pool, classifier)."""
    L = _lib.lib()
    for blk, dims, k in ((MBConv(8, 4, 0.25), TensorDims(128, 14, 14, 128), None),
                         (MBConv(8, 4, 0.25), TensorDims(128, 7, 7, 128), None),
                         (MBConv(8, 4, 0.25, 2), TensorDims(128, 28, 28, 48), 128),
                         (ConvFirst(8, 6), TensorDims(8, 28, 28, 48), None),
                         (ConvFirst(8, 6, 2), TensorDims(8, 56, 56, 32), 48)):
        d = _desc(blk, dims, k)
        assert L.wl_kernel_launches(ctypes.byref(d)) == 1
    d = _desc(Head(1280, 1000), TensorDims(128, 7, 7, 128))
    assert L.wl_kernel_launches(ctypes.byref(d)) == 2


@pytest.mark.parametrize(
    "block,dims,out",
    [
        ("ffn", TensorDims(2, 14, 14, 384), (2, 14, 14, 384)),
        ("patch", TensorDims(2, 224, 224, 3), (2, 56, 56, 96)),
        ("down", TensorDims(2, 56, 56, 96), (2, 28, 28, 192)),
        ("lnhead", TensorDims(3, 7, 7, 768), (3, 1, 1, 1000)),
        ("wide", TensorDims(2, 14, 14, 384), (2, 14, 14, 384)),
    ],
)
def test_convnext_units_descriptors_without_gpu(block, dims, out):
    """The ConvNeXt-T / FFN kinds validate, size their packed blobs and
    workspaces and report output geometry through the ABI on a CPU-only host."""
    from paper_2404_03617_b200.core import FFN, ConvNeXtBlock, Downsample, LNHead, PatchifyStem

    blk = {"ffn": FFN(4, "gelu"), "patch": PatchifyStem(96), "down": Downsample(192), "lnhead": LNHead(1000),
           "wide": ConvNeXtBlock(7, 4, "gelu")}[block]
    s = build_schedule(blk, dims)
    d = block_descriptor(blk, dims, s.out_channels)
    L = _lib.lib()
    assert L.wl_validate(ctypes.byref(d)) == 0
    n, h, w, c = (ctypes.c_int32() for _ in range(4))
    assert L.wl_output_dims(ctypes.byref(d), *(ctypes.byref(v) for v in (n, h, w, c))) == 0
    assert (n.value, h.value, w.value, c.value) == out
    assert L.wl_packed_bytes(ctypes.byref(d)) > 0 and L.wl_workspace_bytes(ctypes.byref(d)) > 4096
    assert L.wl_weight_count(ctypes.byref(d)) == len(weight_names(s))
    for i, name in enumerate(weight_names(s)):
        assert L.wl_weight_numel(ctypes.byref(d), i) == int(np.prod(s.tensor(name).dims))
    packed = _lib.pack_weights(d, [np.ones(s.tensor(nm).dims, np.float32) for nm in weight_names(s)])
    assert packed.nbytes == L.wl_packed_bytes(ctypes.byref(d))


@pytest.mark.parametrize(
    "block,dims,launches",
    [
        (ConvFirst(8, 6), TensorDims(2, 28, 28, 48), 3),
        (MBConv(8, 4, 0.25), TensorDims(4, 14, 14, 128), 5),
        (MBConv(1, 4, 0.25), TensorDims(2, 28, 28, 80), 5),
    ],
)
def test_layer_wise_descriptors_without_gpu(block, dims, launches):
    """WL_SCHEME_LAYER_WISE binds the reference's layer-by-layer schedule
    (one launch per layer, intermediates through the workspace in HBM)."""
    L = _lib.lib()
    s = build_schedule(block, dims, ExecutionScheme.LAYER_WISE)
    d = block_descriptor(block, dims, s.out_channels)
    d.scheme = _lib.SCHEME_LAYER_WISE
    assert L.wl_validate(ctypes.byref(d)) == 0
    assert L.wl_kernel_launches(ctypes.byref(d)) == launches
    m = dims.n * dims.h * dims.w
    hid = block.expansion * dims.c
    assert L.wl_workspace_bytes(ctypes.byref(d)) >= m * hid * 2  # the hidden tensor lives in HBM
    ins = random_inputs(s, np.random.default_rng(1))
    w = [ins[n] for n in weight_names(s)]
    a = _lib.pack_weights(d, w)
    assert a.nbytes == L.wl_packed_bytes(ctypes.byref(d)) and np.array_equal(a, _lib.pack_weights(d, w))


def test_layer_wise_refuses_what_the_reference_does_not_schedule():
    L = _lib.lib()
    for blk, dims, k in ((ConvFirst(8, 6, 2), TensorDims(2, 56, 56, 32), 48),
                         (MBConv(8, 4, 0.25, 2), TensorDims(2, 28, 28, 48), 128),
                         (Stem(16), TensorDims(2, 32, 32, 3), 16)):
        s = build_schedule(blk, dims, out_channels=k)
        d = block_descriptor(blk, dims, s.out_channels)
        d.scheme = _lib.SCHEME_LAYER_WISE
        assert L.wl_validate(ctypes.byref(d)) != 0
    d = _desc(ConvFirst(8, 6), TensorDims(2, 28, 28, 48))
    d.scheme = 7
    assert L.wl_validate(ctypes.byref(d)) == _lib.lib().wl_validate(ctypes.byref(d)) != 0


def test_wide_convfirst_descriptors_without_gpu():
    """Conv-first blocks past the fused kernel's width (C > 128) validate and
    plan three launches: grouped conv + two FFN GEMMs."""
    L = _lib.lib()
    for blk, dims in ((ConvFirst(8, 6), TensorDims(2, 28, 28, 192)), (ConvFirst(1, 4), TensorDims(2, 14, 14, 384))):
        s = build_schedule(blk, dims)
        d = block_descriptor(blk, dims, s.out_channels)
        assert L.wl_validate(ctypes.byref(d)) == 0
        assert L.wl_kernel_launches(ctypes.byref(d)) == 3
        ins = random_inputs(s, np.random.default_rng(0))
        a = _lib.pack_weights(d, [ins[n] for n in weight_names(s)])
        assert a.nbytes == L.wl_packed_bytes(ctypes.byref(d)) and a.any()
