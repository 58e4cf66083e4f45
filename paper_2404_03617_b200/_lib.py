"""ctypes binding of libwlfuse.so (the C ABI in include/wlfuse.h).

The library is built in-tree (``paper_2404_03617_b200/libwlfuse.so``) by
``__graft_entry__.build()``. There is no fallback: if the library or a GPU is
missing, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from functools import lru_cache

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WLFUSE_LIB_AB") or os.path.join(HERE, "libwlfuse.so")  # A/B timing override (tools/ab_build.sh)

WL_OK, WL_EINVAL, WL_EUNSUPPORTED, WL_ECUDA = 0, -1, -2, -3
KIND_CONVFIRST, KIND_MBCONV, KIND_FFN, KIND_STEM, KIND_HEAD = 1, 2, 3, 4, 5
KIND_PATCH_STEM, KIND_DOWNSAMPLE, KIND_LN_HEAD = 6, 7, 8
ACTS = {"identity": 0, "relu": 1, "silu": 2, "sigmoid": 3, "gelu": 4}
NORM_NONE, NORM_LAYERNORM = 0, 1
DTYPE_F16, DTYPE_BF16 = 0, 1
SCHEME_FUSED, SCHEME_LAYER_WISE = 0, 1

# every symbol include/wlfuse.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "wl_version",
    "wl_last_error",
    "wl_init",
    "wl_validate",
    "wl_weight_count",
    "wl_weight_numel",
    "wl_packed_bytes",
    "wl_pack_weights",
    "wl_workspace_bytes",
    "wl_kernel_launches",
    "wl_block_forward",
    "wl_convfirst_fwd",
    "wl_mbconv_fwd",
    "wl_stem_fwd",
    "wl_head_fwd",
    "wl_ffn_fwd",
    "wl_patch_stem_fwd",
    "wl_downsample_fwd",
    "wl_ln_head_fwd",
    "wl_execute_numeric",
    "wl_gemm",
    "wl_stage_forward",
    "wl_stage_max_blocks",
    "wl_pair_supported",
    "wl_pair_packed_bytes",
    "wl_pair_pack",
    "wl_pair_forward",
    "wl_output_dims",
    "wl_debug_set_trace",
)


class BlockDesc(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("n", ctypes.c_int32),
        ("h", ctypes.c_int32),
        ("w", ctypes.c_int32),
        ("c", ctypes.c_int32),
        ("k", ctypes.c_int32),
        ("expansion", ctypes.c_int32),
        ("group_width", ctypes.c_int32),
        ("ksize", ctypes.c_int32),
        ("stride", ctypes.c_int32),
        ("se_sq", ctypes.c_int32),
        ("norm", ctypes.c_int32),
        ("act", ctypes.c_int32),
        ("ln_eps", ctypes.c_float),
        ("embed", ctypes.c_int32),
        ("classes", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("scheme", ctypes.c_int32),
        ("reserved", ctypes.c_int32 * 2),
    ]

    def as_tuple(self):
        return tuple(getattr(self, f) for f, _ in self._fields_[:-1])


class LibraryMissing(RuntimeError):
    pass


class WlError(RuntimeError):
    def __init__(self, code: int, message: str):
        self.code = code
        super().__init__(message)


@lru_cache(maxsize=1)
def lib() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise LibraryMissing(
            f"{LIB_PATH} is not built; run __graft_entry__.build() (there is no CPU fallback)"
        )
    so = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    D = P(BlockDesc)
    vp = ctypes.c_void_p
    sig = {
        "wl_version": (ctypes.c_int, []),
        "wl_last_error": (ctypes.c_char_p, []),
        "wl_init": (ctypes.c_int, [ctypes.c_int]),
        "wl_validate": (ctypes.c_int, [D]),
        "wl_weight_count": (ctypes.c_int, [D]),
        "wl_weight_numel": (ctypes.c_int64, [D, ctypes.c_int]),
        "wl_packed_bytes": (ctypes.c_int64, [D]),
        "wl_pack_weights": (ctypes.c_int, [D, P(P(ctypes.c_float)), ctypes.c_int, vp]),
        "wl_workspace_bytes": (ctypes.c_int64, [D]),
        "wl_kernel_launches": (ctypes.c_int, [D]),
        "wl_block_forward": (ctypes.c_int, [D, vp, vp, vp, vp, vp]),
        "wl_convfirst_fwd": (ctypes.c_int, [D, vp, vp, vp, vp, vp]),
        "wl_mbconv_fwd": (ctypes.c_int, [D, vp, vp, vp, vp, vp]),
        "wl_stem_fwd": (ctypes.c_int, [D, vp, vp, vp, vp, vp]),
        "wl_head_fwd": (ctypes.c_int, [D, vp, vp, vp, vp, vp]),
        "wl_ffn_fwd": (ctypes.c_int, [D, vp, vp, vp, vp, vp]),
        "wl_patch_stem_fwd": (ctypes.c_int, [D, vp, vp, vp, vp, vp]),
        "wl_downsample_fwd": (ctypes.c_int, [D, vp, vp, vp, vp, vp]),
        "wl_ln_head_fwd": (ctypes.c_int, [D, vp, vp, vp, vp, vp]),
        "wl_execute_numeric": (
            ctypes.c_int,
            [D, P(ctypes.c_float), P(P(ctypes.c_float)), ctypes.c_int, P(ctypes.c_float)],
        ),
        "wl_output_dims": (ctypes.c_int, [D] + [P(ctypes.c_int32)] * 4),
        "wl_stage_forward": (ctypes.c_int, [D, ctypes.c_int, vp, P(vp), vp, vp, vp]),
        "wl_stage_max_blocks": (ctypes.c_int, [D]),
        "wl_pair_supported": (ctypes.c_int, [D, D]),
        "wl_pair_packed_bytes": (ctypes.c_int64, [D, D]),
        "wl_pair_pack": (ctypes.c_int, [D, D, P(P(ctypes.c_float)), ctypes.c_int, P(P(ctypes.c_float)), ctypes.c_int, vp]),
        "wl_pair_forward": (ctypes.c_int, [D, D, vp, vp, vp, vp]),
        "wl_gemm": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, vp,
                                   ctypes.c_int, vp, ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, vp]),
        "wl_debug_set_trace": (None, [vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(so, name)
        fn.restype = res
        fn.argtypes = args
    return so


def last_error() -> str:
    return lib().wl_last_error().decode(errors="replace")


def check(code: int, what: str = "") -> int:
    """Map a negative ABI status to the reference's exception types."""
    if code >= 0:
        return code
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if code == WL_EINVAL:
        raise ValueError(msg)
    if code == WL_EUNSUPPORTED:
        from .machine import ScheduleError

        raise ScheduleError(msg)
    raise WlError(code, msg)


def float_ptr_array(arrays):
    """Keep-alive list of contiguous float32 arrays + a float** to them."""
    keep = [np.ascontiguousarray(a, dtype=np.float32) for a in arrays]
    ptrs = (ctypes.POINTER(ctypes.c_float) * len(keep))(
        *[a.ctypes.data_as(ctypes.POINTER(ctypes.c_float)) for a in keep]
    )
    return keep, ptrs


def output_dims(desc: BlockDesc):
    n, h, w, c = (ctypes.c_int32() for _ in range(4))
    check(lib().wl_output_dims(ctypes.byref(desc), *(ctypes.byref(v) for v in (n, h, w, c))), "wl_output_dims")
    return n.value, h.value, w.value, c.value


def pack_weights(desc: BlockDesc, weights) -> np.ndarray:
    """Pack reference float32 tensors (reference order) into the device blob."""
    L = lib()
    check(L.wl_validate(ctypes.byref(desc)), "wl_validate")
    count = check(L.wl_weight_count(ctypes.byref(desc)))
    if len(weights) != count:
        raise ValueError(f"expected {count} weight tensors, got {len(weights)}")
    for i, wt in enumerate(weights):
        want = L.wl_weight_numel(ctypes.byref(desc), i)
        if int(np.size(wt)) != want:
            raise ValueError(f"weight tensor {i} has {np.size(wt)} elements, expected {want}")
    nbytes = check(L.wl_packed_bytes(ctypes.byref(desc)))
    out = np.zeros(nbytes, dtype=np.uint8)
    keep, ptrs = float_ptr_array(weights)
    check(L.wl_pack_weights(ctypes.byref(desc), ptrs, len(keep), out.ctypes.data_as(ctypes.c_void_p)), "pack")
    return out


def execute_numeric_host(desc: BlockDesc, x: np.ndarray, weights) -> np.ndarray:
    """Host-buffer forward through the ABI (H2D, launch, D2H inside)."""
    L = lib()
    n, h, w, c = output_dims(desc)
    out = np.empty((n, h, w, c), dtype=np.float32)
    xk = np.ascontiguousarray(x, dtype=np.float32)
    keep, ptrs = float_ptr_array(weights)
    check(
        L.wl_execute_numeric(
            ctypes.byref(desc),
            xk.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
            ptrs,
            len(keep),
            out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
        ),
        "wl_execute_numeric",
    )
    return out


def gemm(a, b, bias=None, act: str = "identity", res=None, out=None, stream=None):
    """D = act(a @ b.T + bias) (+ res) on the device through ``wl_gemm``:
    a (M, K), b (N, K), res / out (M, N) fp16 or bf16 CUDA tensors (one
    dtype, row-major, contiguous), bias fp32 (N,) or None."""
    import torch

    m, k = a.shape
    n = b.shape[0]
    if a.dtype not in (torch.float16, torch.bfloat16) or b.dtype != a.dtype:
        raise ValueError("wl_gemm takes fp16 or bf16 operands of one dtype")
    dt = DTYPE_BF16 if a.dtype == torch.bfloat16 else DTYPE_F16
    if out is None:
        out = torch.empty((m, n), dtype=a.dtype, device=a.device)
    st = (stream or torch.cuda.current_stream()).cuda_stream
    check(lib().wl_gemm(a.data_ptr(), m, k, a.stride(0), b.data_ptr(), n, b.stride(0), out.data_ptr(), out.stride(0),
                        bias.data_ptr() if bias is not None else None, ACTS[act],
                        res.data_ptr() if res is not None else None, res.stride(0) if res is not None else 0, dt, st),
          "wl_gemm")
    return out
