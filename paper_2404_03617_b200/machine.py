"""Drop-in for the reference tensor machine's execution API
(``waterline.machine``): ``build_schedule`` / ``execute_numeric`` /
``random_inputs`` with the reference's argument meaning, tensor names,
layouts and error types — but ``execute_numeric`` runs the fused sm_100a
kernel of the block through the C ABI (libwlfuse.so) instead of
interpreting a schedule in numpy.

There is no CPU path: without the library or a GPU every call raises.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from .core import (
    BlockSpec,
    ConvFirst,
    ConvNeXtBlock,
    DeviceSpec,
    Downsample,
    ExecutionScheme,
    FFN,
    Head,
    LNHead,
    MBConv,
    PatchifyStem,
    StageSpec,
    Stem,
    TensorDims,
)


class ScheduleError(ValueError):  # machine.py:59-66
    """A schedule violated its construction or execution rules."""

    def __init__(self, message, node=None):
        self.node = node
        if node is not None:
            message = f"node {node}: {message}"
        super().__init__(message)


@dataclass(frozen=True)
class TensorEntry:
    name: str
    dims: tuple[int, ...]
    role: str  # input | weights | output


@dataclass(frozen=True)
class FusedSchedule:
    """A block bound to input dims, carrying the reference's DRAM tensor
    table (names, shapes, order of machine.py:402-415 / 572-590) — what
    ``build_schedule`` returns here."""

    label: str
    scheme: ExecutionScheme
    block: BlockSpec
    dims: TensorDims
    out_channels: int
    tensors: tuple[TensorEntry, ...]
    output: str = "z"
    executable: bool = True
    processors: int | None = None  # the reference's partitioned schedules (same values, machine.py:528-569, 649-660)

    def tensor(self, name: str) -> TensorEntry:
        for t in self.tensors:
            if t.name == name:
                return t
        raise KeyError(name)

    @property
    def out_dims(self) -> tuple[int, ...]:
        return self.tensor("z").dims


def tensor_table(block, dims: TensorDims, k: int) -> tuple[TensorEntry, ...]:
    """DRAM input/weight tensors in the reference's tensor-table order."""
    n, h, w, c = dims.n, dims.h, dims.w, dims.c
    x = TensorEntry("x", (n, h, w, c), "input")
    stride = getattr(block, "stride", 1)
    if isinstance(block, FFN):  # machine.py:345-351
        hid = block.expansion * c
        p = dims.pixels
        return (
            TensorEntry("x", (p, c), "input"),
            TensorEntry("u", (c, hid), "weights"),
            TensorEntry("a", (hid,), "weights"),
            TensorEntry("v", (hid, c), "weights"),
            TensorEntry("b", (c,), "weights"),
            TensorEntry("z", (p, c), "output"),
        )
    out = TensorEntry("z", (n, h // stride, w // stride, k), "output")
    if isinstance(block, ConvFirst):  # machine.py:402-415
        hid = block.expansion * c
        t = block.group_width
        return (
            x,
            TensorEntry("w_conv", (c, 3, 3, t), "weights"),
            TensorEntry("b_conv", (c,), "weights"),
            TensorEntry("u", (c, hid), "weights"),
            TensorEntry("a", (hid,), "weights"),
            TensorEntry("v", (hid, k), "weights"),
            TensorEntry("b", (k,), "weights"),
            out,
        )
    if isinstance(block, ConvNeXtBlock):  # extension: LN affine after the conv
        hid = block.expansion * c
        ks = block.kernel_size
        return (
            x,
            TensorEntry("w_conv", (c, ks, ks, 1), "weights"),
            TensorEntry("b_conv", (c,), "weights"),
            TensorEntry("ln_gamma", (c,), "weights"),
            TensorEntry("ln_beta", (c,), "weights"),
            TensorEntry("u", (c, hid), "weights"),
            TensorEntry("a", (hid,), "weights"),
            TensorEntry("v", (hid, c), "weights"),
            TensorEntry("b", (c,), "weights"),
            out,
        )
    if isinstance(block, MBConv):  # machine.py:572-590
        hid = block.expansion * c
        sq = int(block.se_ratio * c)
        t = block.group_width
        return (
            x,
            TensorEntry("w_exp", (c, hid), "weights"),
            TensorEntry("b_exp", (hid,), "weights"),
            TensorEntry("w_conv", (hid, 3, 3, t), "weights"),
            TensorEntry("b_conv", (hid,), "weights"),
            TensorEntry("w_sq", (hid, sq), "weights"),
            TensorEntry("b_sq", (sq,), "weights"),
            TensorEntry("w_ex", (sq, hid), "weights"),
            TensorEntry("b_ex", (hid,), "weights"),
            TensorEntry("w_prj", (hid, k), "weights"),
            TensorEntry("b_prj", (k,), "weights"),
            out,
        )
    if isinstance(block, PatchifyStem):  # extension (ConvNeXt-T): p x p stride-p conv + LayerNorm
        cs, pt = block.out_channels, block.patch
        return (
            x,
            TensorEntry("w_stem", (cs, pt, pt, c), "weights"),
            TensorEntry("b_stem", (cs,), "weights"),
            TensorEntry("ln_gamma", (cs,), "weights"),
            TensorEntry("ln_beta", (cs,), "weights"),
            TensorEntry("z", (n, h // pt, w // pt, cs), "output"),
        )
    if isinstance(block, Downsample):  # extension (ConvNeXt-T): LayerNorm + 2x2 stride-2 conv
        return (
            x,
            TensorEntry("ln_gamma", (c,), "weights"),
            TensorEntry("ln_beta", (c,), "weights"),
            TensorEntry("w_down", (k, 2, 2, c), "weights"),
            TensorEntry("b_down", (k,), "weights"),
            TensorEntry("z", (n, h // 2, w // 2, k), "output"),
        )
    if isinstance(block, LNHead):  # extension (ConvNeXt-T): pool + LayerNorm + classifier
        m = block.num_classes
        return (
            x,
            TensorEntry("ln_gamma", (c,), "weights"),
            TensorEntry("ln_beta", (c,), "weights"),
            TensorEntry("w_cls", (c, m), "weights"),
            TensorEntry("b_cls", (m,), "weights"),
            TensorEntry("z", (n, m), "output"),
        )
    if isinstance(block, Stem):  # extension: dense 3x3 stride 2 (core.py:135-141)
        cs = block.out_channels
        return (
            x,
            TensorEntry("w_stem", (cs, 3, 3, c), "weights"),
            TensorEntry("b_stem", (cs,), "weights"),
            TensorEntry("z", (n, h // 2, w // 2, cs), "output"),
        )
    if isinstance(block, Head):  # extension: 1x1 conv, pool, classifier (core.py:144-152)
        e, m = block.embed_channels, block.num_classes
        return (
            x,
            TensorEntry("w_embed", (c, e), "weights"),
            TensorEntry("b_embed", (e,), "weights"),
            TensorEntry("w_cls", (e, m), "weights"),
            TensorEntry("b_cls", (m,), "weights"),
            TensorEntry("z", (n, m), "output"),
        )
    raise ValueError(f"{type(block).__name__} blocks have no tensor-machine schedule")


def build_schedule(
    block: BlockSpec,
    dims: TensorDims,
    scheme: ExecutionScheme = ExecutionScheme.BLOCK_FUSION,
    out_channels: int | None = None,
    element_bytes: int = 2,
    chunk: int | None = None,
    processors: int | None = None,
) -> FusedSchedule:
    """Same contract as machine.build_schedule (machine.py:736-772). Both
    schemes build (their traffic is accounted by ``simulate_traffic``) and
    execute on the B200: BLOCK_FUSION on the fused block kernels, LAYER_WISE
    (ConvFirst / MBConv stride 1, FFN) as one launch per layer with every
    intermediate through HBM (layerwise.cu). ``chunk`` / ``processors`` follow the reference's
    validity rules; the fused kernel computes the same values whatever the
    partition (its hidden-chunk widths and CTA split come from the TMEM /
    shared-memory budget)."""
    if not isinstance(block, (FFN, ConvFirst, ConvNeXtBlock, MBConv, Stem, Head, PatchifyStem, Downsample, LNHead)):
        raise ValueError(f"{type(block).__name__} blocks have no tensor-machine schedule")
    k = out_channels if out_channels is not None else dims.c
    if isinstance(block, (Stem, PatchifyStem, Downsample)):
        k = block.out_channels
    elif isinstance(block, (Head, LNHead)):
        k = block.num_classes
    elif getattr(block, "stride", 1) == 1 and k != dims.c:
        raise ValueError("stride-1 blocks keep their channel count")
    if chunk is not None:
        hid = getattr(block, "expansion", 1) * dims.c
        if not 1 <= chunk <= hid or hid % chunk:
            raise ValueError(f"chunk {chunk} does not divide {hid} hidden channels")
    if not processors:  # the reference treats 0 / None as "default partition" (machine.py:655)
        processors = None
    if processors is not None and scheme == ExecutionScheme.BLOCK_FUSION:
        # the reference's partition rules; the B200 kernel computes the same
        # values whatever the partition (its CTA split is planned on chip)
        if isinstance(block, ConvFirst) and processors > 1:  # machine.py:469-474
            if getattr(block, "stride", 1) == 2:
                raise ValueError("the scaling variant models stride-1 blocks only")
            if dims.c % processors or (dims.c // processors) % block.group_width or k != dims.c:
                raise ValueError(f"cannot partition {dims.c} channels across {processors} processors")
        if isinstance(block, MBConv):  # machine.py:655-657
            hid = block.expansion * dims.c
            if processors < 1 or hid % processors or (hid // processors) % block.group_width:
                raise ValueError(f"cannot partition {hid} hidden channels across {processors} processors")
    return FusedSchedule(
        label=f"{block.kind}-{scheme.value}",
        scheme=scheme,
        block=block,
        dims=dims,
        out_channels=k,
        tensors=tensor_table(block, dims, k),
        processors=processors,
    )


def random_inputs(s: FusedSchedule, rng: np.random.Generator, scale: float = 0.5) -> dict:
    """0.5 N(0,1) float32 per DRAM input/weight, in tensor-table order
    (machine.py:1064-1070): the same seed yields the same arrays as the
    reference for the reference's block kinds."""
    return {
        t.name: (scale * rng.standard_normal(t.dims)).astype(np.float32)
        for t in s.tensors
        if t.role in ("input", "weights")
    }


def block_descriptor(block, dims: TensorDims, k: int):
    """The C-ABI descriptor (include/wlfuse.h) of a block bound to dims."""
    from . import _lib

    d = _lib.BlockDesc()
    d.n, d.h, d.w, d.c, d.k = dims.n, dims.h, dims.w, dims.c, k
    d.ln_eps = 1e-6
    if isinstance(block, ConvFirst):
        d.kind = _lib.KIND_CONVFIRST
        d.expansion, d.group_width, d.ksize, d.stride = block.expansion, block.group_width, 3, block.stride
        d.act = _act(block.activation)
    elif isinstance(block, ConvNeXtBlock):
        d.kind = _lib.KIND_CONVFIRST
        d.expansion, d.group_width, d.ksize, d.stride = block.expansion, 1, block.kernel_size, 1
        d.norm, d.ln_eps = _lib.NORM_LAYERNORM, block.layer_norm_eps
        d.act = _act(block.activation)
    elif isinstance(block, MBConv):
        d.kind = _lib.KIND_MBCONV
        d.expansion, d.group_width, d.ksize, d.stride = block.expansion, block.group_width, 3, block.stride
        d.se_sq = int(block.se_ratio * dims.c)
        d.act = _act(block.activation)
    elif isinstance(block, FFN):
        d.kind = _lib.KIND_FFN
        d.expansion = block.expansion
        d.act = _act(block.activation)
    elif isinstance(block, PatchifyStem):
        d.kind = _lib.KIND_PATCH_STEM
        d.k, d.ksize, d.stride = block.out_channels, block.patch, block.patch
        d.norm, d.ln_eps = _lib.NORM_LAYERNORM, block.layer_norm_eps
    elif isinstance(block, Downsample):
        d.kind = _lib.KIND_DOWNSAMPLE
        d.k, d.ksize, d.stride = block.out_channels, 2, 2
        d.norm, d.ln_eps = _lib.NORM_LAYERNORM, block.layer_norm_eps
    elif isinstance(block, LNHead):
        d.kind = _lib.KIND_LN_HEAD
        d.classes, d.k = block.num_classes, block.num_classes
        d.norm, d.ln_eps = _lib.NORM_LAYERNORM, block.layer_norm_eps
    elif isinstance(block, Stem):
        d.kind = _lib.KIND_STEM
        d.k, d.stride, d.ksize = block.out_channels, 2, 3
        d.act = _act(block.activation)
    elif isinstance(block, Head):
        d.kind = _lib.KIND_HEAD
        d.embed, d.classes, d.k = block.embed_channels, block.num_classes, block.num_classes
        d.act = _act("relu")
    else:
        raise ScheduleError(f"{type(block).__name__} has no B200 fused kernel")
    return d


def device_channels(c: int) -> int:
    """Channel count a block boundary runs at on the device: the kernels'
    K-steps and channel-pair tiles need C % 16 == 0, so ConvFirstNet-Nano's
    24 and Tiny's 72 run as 32 and 80. The extra channels are exact zeros
    end to end (zero weights and biases; ReLU/SiLU/GELU(0) = 0; the SE gate
    of a zero channel multiplies zero), so the real channels are unchanged."""
    return c if c % 16 == 0 else -(-c // 16) * 16


_SQ_AXIS = {"w_sq": 1, "b_sq": 0, "w_ex": 0}  # SE squeeze width stays the real int(se_ratio * C)


@dataclass(frozen=True)
class DeviceBinding:
    """A schedule (reference shapes) bound to its device channel counts:
    the C-ABI descriptor plus the zero-embedding of reference-shaped
    weights and activations into the padded device tensors."""

    schedule: FusedSchedule
    block: object  # the block as the device runs it (a Stem carries its padded width)
    dims: TensorDims  # device input dims
    k: int  # device output channels
    desc: object

    @property
    def padded(self) -> bool:
        return self.dims.c != self.schedule.dims.c or self.k != self.schedule.out_channels

    @property
    def out_dims(self) -> tuple[int, ...]:
        d = self.schedule.out_dims
        return d if len(d) == 2 else (*d[:3], self.k)

    def device_weights(self, weights: dict) -> list[np.ndarray]:
        """Reference-named float32 weights -> the device list (padded)."""
        dev = build_schedule(self.block, self.dims, out_channels=self.k)
        out = []
        for t in self.schedule.tensors:
            if t.role != "weights":
                continue
            w = np.asarray(weights[t.name], dtype=np.float32)
            if w.shape != t.dims:
                raise ScheduleError(f"weight {t.name!r} has shape {w.shape}, expected {t.dims}")
            if not self.padded:
                out.append(w)
                continue
            shape = list(dev.tensor(t.name).dims)
            if t.name in _SQ_AXIS:
                shape[_SQ_AXIS[t.name]] = t.dims[_SQ_AXIS[t.name]]
            z = np.zeros(shape, dtype=np.float32)
            z[tuple(slice(0, n) for n in w.shape)] = w
            out.append(z)
        return out

    def device_input(self, x: np.ndarray) -> np.ndarray:
        if x.shape[-1] == self.dims.c:
            return x
        z = np.zeros((*x.shape[:-1], self.dims.c), dtype=x.dtype)
        z[..., : x.shape[-1]] = x
        return z

    def real_output(self, z):
        """Device output -> the reference's channel count (a view)."""
        return z if len(self.schedule.out_dims) == 2 else z[..., : self.schedule.out_channels]


def device_binding(s: FusedSchedule) -> DeviceBinding:
    block, dims = s.block, s.dims
    if isinstance(block, (FFN, PatchifyStem, Downsample, LNHead)):
        # row-wise units (FFN rows, LayerNorm units): run at the reference widths (C % 8 == 0)
        if dims.c % 8 and not isinstance(block, PatchifyStem):
            raise ScheduleError(f"{type(block).__name__} needs C % 8 == 0 on the device (C = {dims.c})")
        return DeviceBinding(s, block, dims, s.out_channels, block_descriptor(block, dims, s.out_channels))
    cin = dims.c if isinstance(block, Stem) else device_channels(dims.c)
    k = s.out_channels if isinstance(block, Head) else device_channels(s.out_channels)
    if isinstance(block, ConvNeXtBlock) and cin != dims.c:
        raise ScheduleError("LayerNorm blocks cannot be zero-padded (the padding would enter the channel mean)")
    ddims = TensorDims(dims.n, dims.h, dims.w, cin)
    dblock = replace(block, out_channels=k) if isinstance(block, Stem) else block
    desc = block_descriptor(dblock, ddims, k)
    if isinstance(block, MBConv):
        desc.se_sq = int(block.se_ratio * dims.c)
    return DeviceBinding(s, dblock, ddims, k, desc)


def _act(name: str) -> int:
    from . import _lib

    if name not in _lib.ACTS:
        raise ValueError(f"unknown activation {name!r}")
    return _lib.ACTS[name]


def weight_names(s: FusedSchedule) -> list[str]:
    return [t.name for t in s.tensors if t.role == "weights"]


def execute_numeric(s: FusedSchedule, inputs: dict) -> np.ndarray:
    """Fused-kernel evaluation with execute_numeric's contract
    (machine.py:1053-1061): float32 inputs keyed by tensor name, float32
    output; missing or mis-shaped inputs raise ScheduleError. Inputs are
    rounded to fp16 on the way in (the kernels' storage type), accumulation
    is fp32 in TMEM, and the result is the fp16 output widened to float32.
    LAYER_WISE schedules run the reference's layer-by-layer order
    (machine.py:418-459, 593-646, 339-365) as separate device launches."""
    layer_wise = s.scheme == ExecutionScheme.LAYER_WISE
    if layer_wise and not isinstance(s.block, (ConvFirst, MBConv, FFN)):
        raise ScheduleError(f"the reference has no layer-wise schedule for {type(s.block).__name__} units")
    arrays = {}
    for t in s.tensors:
        if t.role not in ("input", "weights"):
            continue
        if t.name not in inputs:
            raise ScheduleError(f"missing input tensor {t.name!r}")
        arr = np.asarray(inputs[t.name], dtype=np.float32)
        if arr.shape != t.dims:
            raise ScheduleError(f"input {t.name!r} has shape {arr.shape}, expected {t.dims}")
        arrays[t.name] = arr
    from . import _lib

    b = device_binding(s)
    if layer_wise:
        b.desc.scheme = _lib.SCHEME_LAYER_WISE
    out = _lib.execute_numeric_host(b.desc, b.device_input(arrays["x"]), b.device_weights(arrays))
    return np.ascontiguousarray(b.real_output(out.reshape(b.out_dims)))


def fused_dram_bytes(s: FusedSchedule, element_bytes: int = 2) -> int:
    """The tensor-machine DRAM plan of the fused kernel (simulate_traffic of
    the BLOCK_FUSION schedule, machine.py:826-869 == complexity.block_costs)."""
    from . import complexity
    from .core import ExecutionScheme as ES

    dev = DeviceSpec("accounting", 1.0, 1.0, bytes_per_element=element_bytes)
    return complexity.block_costs(s.block, s.dims, ES.BLOCK_FUSION, dev, out_channels=s.out_channels).bytes


# ------------------------------------------------------------ micro-batching


@dataclass(frozen=True)
class MicrobatchPlan:  # machine.py:1077-1088
    feasible: bool
    micro_batch: int
    fusible_depth: int
    activation_bytes: int
    weights_bytes: int
    l2_bytes: int

    @property
    def total_bytes(self) -> int:
        return self.activation_bytes + self.weights_bytes


def microbatch_plan(stage: StageSpec, dims: TensorDims, device: DeviceSpec, conv_taps: int | None = None) -> MicrobatchPlan:
    """Largest (micro-batch, depth) whose activations and weights fit in L2
    (machine.py:1091-1120). ``conv_taps`` generalises the reference's
    hard-coded 72 (= 9 taps x group width 8) weights per hidden channel."""
    if not isinstance(stage.block, MBConv):
        raise ValueError("micro-batch planning applies to MBConv stages")
    if device.l2_bytes <= 0:
        raise ValueError("device has no usable global-memory capacity")
    if dims.c != stage.channels:
        raise ValueError(f"dims carry {dims.c} channels but the stage has {stage.channels}")
    bpe, a, c = device.bytes_per_element, stage.block.expansion, stage.channels
    taps = conv_taps if conv_taps is not None else 72
    per_image = bpe * 2 * dims.h * dims.w * c
    per_block = bpe * (2 * a * c * c + taps * a * c)
    for depth in range(stage.depth, 0, -1):
        budget = device.l2_bytes - depth * per_block
        if budget >= per_image:
            nmb = min(dims.n, budget // per_image)
            return MicrobatchPlan(True, int(nmb), depth, int(nmb) * per_image, depth * per_block, device.l2_bytes)
    return MicrobatchPlan(False, 0, 0, 0, per_block, device.l2_bytes)


# the reference's accounting / FFN helpers (machine.py:228-252, 786-897)
from .traffic import (  # noqa: E402,F401
    TrafficReport,
    dram_bytes_by_role,
    ffn_fused,
    ffn_layerwise,
    simulate_traffic,
    validate_schedule,
)
