"""The tensor machine's accounting API for the schedules ``machine.
build_schedule`` returns: ``simulate_traffic`` (machine.py:826-869),
``dram_bytes_by_role`` (machine.py:872-897) and ``validate_schedule``
(machine.py:786-819), plus the FFN numeric helpers ``ffn_layerwise`` /
``ffn_fused`` (machine.py:228-252).

The reference walks a node list; here every schedule is a tensor table
bound to a block, so the walk is restated per schedule family as the list
of tier crossings it performs: ``(DRAM-side role or None, elements,
crosses DRAM<->GLOBAL, crosses GLOBAL<->LOCAL)``. Each list follows the
reference schedule builder line by line (cited per family); the numbers are
pinned against the unmodified reference on a grid of blocks and shapes
(tests/golden/traffic.json, tests/test_traffic.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import ConvFirst, ConvNeXtBlock, ExecutionScheme, FFN, MBConv


@dataclass(frozen=True)
class TrafficReport:  # machine.py:161-169
    dram_global_bytes: int
    global_local_bytes: int
    mac_ops: int
    sync_count: int

    @property
    def dram_bytes(self) -> int:
        return self.dram_global_bytes


# a crossing: (role of the DRAM-side tensor or None, elements, DRAM<->GLOBAL, GLOBAL<->LOCAL)
_D2L, _D2G, _G2L = (True, True), (True, False), (False, True)


def _chunk_width(hidden: int, group_width: int) -> int:  # machine.py:325-329
    r = min(group_width, hidden)
    while hidden % r:
        r -= 1
    return r


def _partition_count(hidden: int, group_width: int) -> int:  # machine.py:332-336
    for p in (8, 4, 2):
        if hidden % p == 0 and (hidden // p) % group_width == 0:
            return p
    return 1


def _ffn(s):
    n_pix, c = s.dims.pixels, s.dims.c
    hid = s.block.expansion * c
    macs = 2 * n_pix * c * hid
    if s.scheme == ExecutionScheme.LAYER_WISE:  # machine.py:255-283
        mv = [("input", n_pix * c, *_D2L), ("weights", c * hid, *_D2L), ("weights", hid, *_D2L),
              ("hidden", n_pix * hid, *_D2L), ("hidden", n_pix * hid, *_D2L),
              ("weights", hid * c, *_D2L), ("weights", c, *_D2L), ("output", n_pix * c, *_D2L)]
        return mv, macs, 0
    # machine.py:286-317: U, a, V staged in GLOBAL, sliced per chunk trip
    mv = [("input", n_pix * c, *_D2L), ("weights", c * hid, *_D2G), ("weights", hid, *_D2G),
          ("weights", hid * c, *_D2G), ("weights", c, *_D2L),
          (None, c * hid + hid + hid * c, *_G2L), ("output", n_pix * c, *_D2L)]
    return mv, macs, 0


def _convfirst(s):
    b, d, k = s.block, s.dims, s.out_channels
    n, h, w, c = d.n, d.h, d.w, d.c
    t = b.group_width if isinstance(b, ConvFirst) else 1
    taps = 9 if isinstance(b, ConvFirst) else b.kernel_size ** 2
    hid = b.expansion * c
    nhw = n * h * w
    s2 = getattr(b, "stride", 1) == 2
    x_el, wc_el = nhw * c, c * taps * t
    extra = [("weights", c, *_D2L), ("weights", c, *_D2L)] if isinstance(b, ConvNeXtBlock) else []
    conv_macs = nhw * c * taps * t
    if s.scheme == ExecutionScheme.LAYER_WISE:  # machine.py:418-459
        if s2:
            hw2, hw4 = (h * w) // 2, (h * w) // 4
            xc_el, y_st, y_ld, z_el = n * hw2 * c, n * hw4 * hid, n * hw4 * hid, n * hw4 * k
            macs = conv_macs + n * hw2 * c * hid + n * hw4 * hid * k
        else:
            xc_el, y_st, y_ld, z_el = nhw * c, nhw * hid, nhw * hid, nhw * k
            macs = conv_macs + nhw * c * hid + nhw * hid * k
        mv = [("input", x_el, *_D2L), ("weights", wc_el, *_D2L), ("weights", c, *_D2L), *extra,
              ("hidden", xc_el, *_D2L), ("hidden", xc_el, *_D2L), ("weights", c * hid, *_D2L),
              ("weights", hid, *_D2L), ("hidden", y_st, *_D2L), ("hidden", y_ld, *_D2L),
              ("weights", hid * k, *_D2L), ("weights", k, *_D2L)]
        if not s2:
            mv.append(("input", x_el, *_D2L))  # the projection re-reads the shortcut
        mv.append(("output", z_el, *_D2L))
        return mv, macs, 0
    p = s.processors or 1
    if p > 1:  # machine.py:528-569: channel partitions meet in GLOBAL, one sync
        macs = conv_macs + nhw * c * hid + nhw * hid * c
        mv = [("weights", hid, *_D2G), ("input", x_el, *_D2L), ("weights", wc_el, *_D2L),
              ("weights", c, *_D2L), *extra, ("weights", c * hid, *_D2L),
              (None, p * nhw * hid, *_G2L), (None, p * nhw * hid, *_G2L), (None, p * hid, *_G2L),
              ("weights", hid * c, *_D2L), ("weights", c, *_D2L), ("output", nhw * c, *_D2L)]
        return mv, macs, 1
    # machine.py:462-525: U, a, V staged in GLOBAL and sliced per chunk trip
    if s2:
        hw2, hw4 = (h * w) // 2, (h * w) // 4
        macs = conv_macs + n * hw2 * c * hid + n * hw4 * hid * k
        z_el = n * hw4 * k
    else:
        macs = conv_macs + nhw * c * hid + nhw * hid * k
        z_el = nhw * k
    mv = [("input", x_el, *_D2L), ("weights", wc_el, *_D2L), ("weights", c, *_D2L), *extra,
          ("weights", c * hid, *_D2G), ("weights", hid, *_D2G), ("weights", hid * k, *_D2G),
          ("weights", k, *_D2L), (None, c * hid + hid + hid * k, *_G2L), ("output", z_el, *_D2L)]
    return mv, macs, 0


def _mbconv(s):
    b, d, k = s.block, s.dims, s.out_channels
    n, h, w, c = d.n, d.h, d.w, d.c
    t, hid = b.group_width, b.expansion * c
    sq = int(b.se_ratio * c)
    nhw = n * h * w
    s2 = b.stride == 2
    rows = n * (h * w) // 4 if s2 else nhw
    macs = nhw * c * hid + nhw * hid * 9 * t + 2 * n * hid * sq + rows * hid * k
    w_el = [c * hid, hid, hid * 9 * t, hid, hid * sq, sq, sq * hid, hid, hid * k, k]
    if s.scheme == ExecutionScheme.LAYER_WISE:  # machine.py:593-646 (SE biases ride along uncounted)
        mv = [("input", nhw * c, *_D2L), ("weights", w_el[0], *_D2L), ("weights", w_el[1], *_D2L),
              ("hidden", nhw * hid, *_D2L), ("hidden", nhw * hid, *_D2L), ("weights", w_el[2], *_D2L),
              ("weights", w_el[3], *_D2L), ("hidden", rows * hid, *_D2L), ("hidden", rows * hid, *_D2L),
              ("weights", w_el[4], *_D2L), ("weights", w_el[6], *_D2L), ("hidden", rows * hid, *_D2L),
              ("hidden", rows * hid, *_D2L), ("weights", w_el[8], *_D2L), ("weights", w_el[9], *_D2L)]
        if not s2:
            mv.append(("input", nhw * c, *_D2L))
        mv.append(("output", rows * k, *_D2L))
        return mv, macs, 0
    # machine.py:649-733: everything staged through GLOBAL once; per partition
    # (parallel trips) the input, weight slices, the squeeze exchange and the
    # accumulation onto the staged input (stride 1) or a GLOBAL accumulator
    p = s.processors or _partition_count(hid, t)
    acc = rows * k if s2 else nhw * c
    mv = [("input", nhw * c, *_D2G)] + [("weights", e, *_D2G) for e in w_el]
    per = nhw * c + (c * hid + hid + hid * 9 * t + hid + hid * sq + sq * hid + hid + hid * k) // p
    per += 2 * n * sq + sq + acc
    mv += [(None, p * per, *_G2L), (None, acc + k, *_G2L), ("output", rows * k, *_D2L)]
    return mv, macs, 1


def _walk(s):
    if isinstance(s.block, FFN):
        return _ffn(s)
    if isinstance(s.block, (ConvFirst, ConvNeXtBlock)):
        return _convfirst(s)
    if isinstance(s.block, MBConv):
        return _mbconv(s)
    raise ValueError(f"{type(s.block).__name__} blocks have no tensor-machine schedule")


def validate_schedule(s) -> None:
    """Static well-formedness (machine.py:786-819): every tensor the block's
    algorithm reads is declared with its reference shape, exactly one output."""
    from .machine import ScheduleError, tensor_table

    want = tensor_table(s.block, s.dims, s.out_channels)
    names = [t.name for t in s.tensors]
    if len(set(names)) != len(names):
        raise ScheduleError("duplicate tensor in the tensor table")
    for t in want:
        if t.name not in names:
            raise ScheduleError(f"undeclared tensor {t.name!r}")
        if s.tensor(t.name).dims != t.dims:
            raise ScheduleError(f"tensor {t.name!r} has dims {s.tensor(t.name).dims}, expected {t.dims}")
    if sum(1 for t in s.tensors if t.role == "output") != 1:
        raise ScheduleError("a schedule writes exactly one output tensor")


def simulate_traffic(s, element_bytes: int = 2) -> TrafficReport:
    """Bytes per tier crossing, MACs (matmul + grouped conv only) and sync
    markers of a schedule (machine.py:826-869)."""
    validate_schedule(s)
    mv, macs, syncs = _walk(s)
    dg = sum(e for _, e, a, _ in mv if a) * element_bytes
    gl = sum(e for _, e, _, g in mv if g) * element_bytes
    return TrafficReport(dg, gl, macs, syncs)


def dram_bytes_by_role(s, element_bytes: int = 2) -> dict[str, int]:
    """DRAM-crossing bytes by the role of the DRAM-side tensor (machine.py:872-897)."""
    validate_schedule(s)
    out: dict[str, int] = {}
    for role, e, _, _ in _walk(s)[0]:
        if role is not None:
            out[role] = out.get(role, 0) + e * element_bytes
    return out


def _check_ffn_shapes(x, u, v, a, b):  # machine.py:214-225
    p, c = x.shape
    hid = u.shape[1]
    if u.shape[0] != c:
        raise ValueError(f"U must be {c}x{hid}, got {u.shape}")
    if v.shape != (hid, c):
        raise ValueError(f"V must be {hid}x{c}, got {v.shape}")
    if a.shape != (hid,):
        raise ValueError(f"a must have {hid} entries, got {a.shape}")
    if b.shape != (c,):
        raise ValueError(f"b must have {c} entries, got {b.shape}")
    return p, c, hid


def _phi(name, v):
    v = np.asarray(v, dtype=np.float64)
    if name == "relu":
        return np.maximum(v, 0.0)
    if name == "silu":
        return v / (1.0 + np.exp(-v))
    if name == "sigmoid":
        return 1.0 / (1.0 + np.exp(-v))
    if name == "identity":
        return v
    raise ValueError(f"unknown activation {name!r}")


def ffn_layerwise(x, u, v, a, b, activation: str = "relu") -> np.ndarray:
    """phi(XU + a)V + b through an explicit fp32 hidden tensor (machine.py:228-233).
    These two helpers are the reference's own host-side definitions of the
    FFN identity the fused kernels implement; the GPU path is
    ``machine.execute_numeric`` on an FFN schedule."""
    x, u, v, a, b = (np.asarray(m) for m in (x, u, v, a, b))
    _check_ffn_shapes(x, u, v, a, b)
    y = _phi(activation, x.astype(np.float64) @ u.astype(np.float64) + a).astype(np.float32)
    return (y.astype(np.float64) @ v.astype(np.float64) + b).astype(np.float32)


def ffn_fused(x, u, v, a, b, activation: str = "relu", chunk: int = 1) -> np.ndarray:
    """Sum over hidden chunks of phi(X U_r + a_r) V_r, + b (machine.py:236-252)."""
    x, u, v, a, b = (np.asarray(m) for m in (x, u, v, a, b))
    _, c, hid = _check_ffn_shapes(x, u, v, a, b)
    if not 1 <= chunk <= hid:
        raise ValueError(f"chunk must lie in [1, {hid}], got {chunk}")
    x64, u64, v64 = x.astype(np.float64), u.astype(np.float64), v.astype(np.float64)
    acc = np.zeros((x.shape[0], c), dtype=np.float64)
    for lo in range(0, hid, chunk):
        sl = slice(lo, min(lo + chunk, hid))
        y = _phi(activation, x64 @ u64[:, sl] + a[sl]).astype(np.float32)
        acc += y.astype(np.float64) @ v64[sl]
    return (acc + b).astype(np.float32)


def chunk_width(block, dims) -> int:
    """Hidden channels per chunk trip of the reference's fused schedule."""
    return _chunk_width(getattr(block, "expansion", 1) * dims.c, getattr(block, "group_width", 8))


def partition_count(block, dims) -> int:
    return _partition_count(block.expansion * dims.c, block.group_width)


__all__ = ["TrafficReport", "simulate_traffic", "dram_bytes_by_role", "validate_schedule", "ffn_layerwise",
           "ffn_fused"]
