"""``torch.nn.Module`` wrappers around the fused kernels (the paper's
TorchBlock pattern), plus the fan-in-scaled synthetic
weight init used for whole-network runs.

Each module owns its packed weights and workspace on the device and launches
its block through the C ABI on the current torch stream. Inputs/outputs are
NHWC fp16 CUDA tensors. No CPU fallback: construction raises without a GPU
or without libwlfuse.so.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .core import ConvFirst, ConvNeXtBlock, ExecutionScheme, Head, MBConv, Stem, TensorDims
from .machine import FusedSchedule, build_schedule, device_binding, random_inputs


def init_weights(s: FusedSchedule, rng: np.random.Generator, residual_gain: float = 0.5) -> dict:
    """Fan-in-scaled weights N(0, 1/fan_in), biases 0.1 N(0, 1), LayerNorm
    gamma 1 + 0.1 N, beta 0.1 N (documented in DESIGN.md: the reference's
    0.5 N(0,1) init overflows fp16 after three chained blocks). Projections
    feeding a residual are scaled by ``residual_gain``."""
    out = {}
    block = s.block
    for t in s.tensors:
        if t.role != "weights":
            continue
        name, dims = t.name, t.dims
        if len(dims) == 1:
            if name == "ln_gamma":
                out[name] = (1.0 + 0.1 * rng.standard_normal(dims)).astype(np.float32)
            else:
                out[name] = (0.1 * rng.standard_normal(dims)).astype(np.float32)
            continue
        if len(dims) == 4:  # (K, R, S, T): fan-in R*S*T
            fan_in = dims[1] * dims[2] * dims[3]
        else:  # (in, out) matrices
            fan_in = dims[0]
        w = rng.standard_normal(dims) / np.sqrt(fan_in)
        if name in ("v", "w_prj") and getattr(block, "stride", 1) == 1 and not isinstance(block, (Stem, Head)):
            w = w * residual_gain
        out[name] = w.astype(np.float32)
    return out


class FusedBlock(torch.nn.Module):
    """One fused block bound to a batch geometry (the layer of the
    model-level scheduler). ``weights`` uses the reference tensor names.
    ``scheme=LAYER_WISE`` binds the same block to the reference's layer-wise
    schedule (one launch per layer, intermediates through HBM) — the
    baseline the fused kernels are compared with."""

    def __init__(self, block, dims: TensorDims, out_channels: int | None = None, weights: dict | None = None,
                 seed: int = 0, device: str | torch.device = "cuda", dtype: torch.dtype = torch.float16,
                 scheme: ExecutionScheme = ExecutionScheme.BLOCK_FUSION):
        super().__init__()
        if not torch.cuda.is_available():
            raise RuntimeError("FusedBlock needs a CUDA device (there is no CPU fallback)")
        if dtype not in (torch.float16, torch.bfloat16):
            raise ValueError("FusedBlock stores activations and weights in fp16 or bf16")
        self.dtype = dtype
        self.schedule = build_schedule(block, dims, scheme=scheme, out_channels=out_channels)
        self.binding = device_binding(self.schedule)  # zero-padded channels where C % 16 != 0
        self.desc = self.binding.desc
        self.desc.dtype = _lib.DTYPE_BF16 if dtype == torch.bfloat16 else _lib.DTYPE_F16
        if scheme == ExecutionScheme.LAYER_WISE:
            self.desc.scheme = _lib.SCHEME_LAYER_WISE
        _lib.check(_lib.lib().wl_validate(ctypes.byref(self.desc)), f"{self.schedule.label} ({dtype})")
        L = _lib.lib()
        dev = torch.device(device)
        _lib.check(L.wl_init(dev.index if dev.index is not None else torch.cuda.current_device()), "wl_init")
        if weights is None:
            weights = init_weights(self.schedule, np.random.default_rng(seed))
        self.weights = {k: np.asarray(v, dtype=np.float32) for k, v in weights.items()}
        packed = _lib.pack_weights(self.desc, self.binding.device_weights(self.weights))
        self.register_buffer("packed", torch.from_numpy(packed).to(dev), persistent=False)
        ws = _lib.check(L.wl_workspace_bytes(ctypes.byref(self.desc)))
        self.register_buffer("workspace", torch.zeros(max(ws, 256), dtype=torch.uint8, device=dev), persistent=False)
        self.out_shape = tuple(self.binding.out_dims)  # device shape (padded channels)
        self.in_shape = (dims.n, dims.h, dims.w, self.binding.dims.c)

    def launch(self, x: torch.Tensor, out: torch.Tensor, workspace: torch.Tensor | None = None, stream=None) -> None:
        """Raw launch into a caller-owned output (graph-capturable). ``x``
        and ``out`` carry the device channel counts (``in_shape`` /
        ``out_shape``; padded channels are zero)."""
        ws = self.workspace if workspace is None else workspace
        st = (stream or torch.cuda.current_stream()).cuda_stream
        _lib.check(
            _lib.lib().wl_block_forward(
                ctypes.byref(self.desc), x.data_ptr(), self.packed.data_ptr(), out.data_ptr(), ws.data_ptr(), st
            ),
            f"{self.schedule.label}",
        )

    def launch_count(self) -> int:
        """Kernel launches one ``launch`` issues (wl_kernel_launches)."""
        return _lib.check(_lib.lib().wl_kernel_launches(ctypes.byref(self.desc)), "wl_kernel_launches")

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if x.dtype != self.dtype or not x.is_cuda or not x.is_contiguous():
            raise ValueError(f"FusedBlock expects a contiguous NHWC {self.dtype} CUDA tensor")
        want = (self.schedule.dims.n, self.schedule.dims.h, self.schedule.dims.w, self.schedule.dims.c)
        if tuple(x.shape) != want:
            raise ValueError(f"input shape {tuple(x.shape)} does not match the bound dims {want}")
        if self.in_shape != want:
            x = torch.nn.functional.pad(x, (0, self.in_shape[3] - want[3]))
        out = torch.empty(self.out_shape, dtype=self.dtype, device=x.device)
        self.launch(x, out)
        return self.binding.real_output(out).contiguous() if self.binding.padded else out


def FusedConvFirst(dims: TensorDims, group_width=8, expansion=6, stride=1, activation="relu", out_channels=None, **kw):
    return FusedBlock(ConvFirst(group_width, expansion, stride, activation), dims, out_channels, **kw)


def FusedConvNeXtBlock(dims: TensorDims, kernel_size=7, expansion=4, activation="gelu", **kw):
    return FusedBlock(ConvNeXtBlock(kernel_size, expansion, activation), dims, None, **kw)


def FusedMBConv(dims: TensorDims, group_width=8, expansion=4, se_ratio=0.25, stride=1, activation="silu",
                out_channels=None, **kw):
    return FusedBlock(MBConv(group_width, expansion, se_ratio, stride, activation), dims, out_channels, **kw)


__all__ = ["FusedBlock", "FusedConvFirst", "FusedConvNeXtBlock", "FusedMBConv", "init_weights", "random_inputs"]
