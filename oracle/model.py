"""Whole-network CPU oracle (TEST INFRASTRUCTURE / CPU baseline only).

Composes the block restatements of ``oracle.blocks`` along the reference's
``plan_blocks`` order (core.py:362-398). Activations are stored in fp16
between units, exactly as the GPU path stores them, so a per-unit parity
check can feed the oracle the GPU's own unit input.
"""

from __future__ import annotations

import numpy as np

from . import blocks as B


def unit_forward(block, weights: dict, x: np.ndarray) -> np.ndarray:
    """One plan_blocks unit on the CPU (float32 result)."""
    kind = block.kind
    w = weights
    if kind == "stem":
        return B.stem_block(x, w["w_stem"], w["b_stem"], block.activation)
    if kind == "head":
        return B.head_block(x, w["w_embed"], w["b_embed"], w["w_cls"], w["b_cls"])
    if kind == "convfirst":
        args = (x, w["w_conv"], w["b_conv"], w["u"], w["a"], w["v"], w["b"])
        if block.stride == 2:
            return B.convfirst_s2_block(*args, activation=block.activation)
        return B.convfirst_block(*args, activation=block.activation)
    if kind == "convnext":
        return B.convnext_block(
            x, w["w_conv"], w["b_conv"], w["u"], w["a"], w["v"], w["b"], activation=block.activation,
            ln_gamma=w["ln_gamma"], ln_beta=w["ln_beta"], ln_eps=block.layer_norm_eps,
        )
    if kind == "patch_stem":
        return B.patch_stem_block(x, w["w_stem"], w["b_stem"], w["ln_gamma"], w["ln_beta"], block.layer_norm_eps)
    if kind == "downsample":
        return B.downsample_block(x, w["ln_gamma"], w["ln_beta"], w["w_down"], w["b_down"], block.layer_norm_eps)
    if kind == "ln_head":
        return B.ln_head_block(x, w["ln_gamma"], w["ln_beta"], w["w_cls"], w["b_cls"], block.layer_norm_eps)
    if kind == "ffn":
        return B.ffn_block(x, w["u"], w["a"], w["v"], w["b"], block.activation)
    if kind == "mbconv":
        return B.mbconv_block(
            x, w["w_exp"], w["b_exp"], w["w_conv"], w["b_conv"], w["w_sq"], w["b_sq"], w["w_ex"], w["b_ex"],
            w["w_prj"], w["b_prj"], activation=block.activation, stride=block.stride,
        )
    raise ValueError(f"no oracle for block kind {kind!r}")


def network_forward(units, weights: dict, x: np.ndarray, fp16_between_units: bool = True) -> np.ndarray:
    """``units``: the plan_blocks list; ``weights``: label -> tensors."""
    h = np.asarray(x, dtype=np.float32)
    for u in units:
        h = unit_forward(u.block, weights[u.label], h)
        if fp16_between_units:
            h = h.astype(np.float16).astype(np.float32)
    return h
