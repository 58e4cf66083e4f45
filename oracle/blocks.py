"""Numpy restatement of the reference block semantics (TEST INFRASTRUCTURE).

Conventions follow the reference tensor machine (``/root/reference/pkg/src/
waterline/machine.py``): tensors are stored in float32 at every layer
boundary, every matmul / convolution accumulates in float64
(machine.py:1009-1043), activations evaluate in float64 (machine.py:178-188).
Each function cites the reference lines it restates; functions marked
UNPINNED have no executable counterpart in the reference.
"""

from __future__ import annotations

import math

import numpy as np

F32, F64 = np.float32, np.float64


def _f32(a) -> np.ndarray:
    return np.asarray(a, dtype=F64).astype(F32)


def phi(name: str, x) -> np.ndarray:
    """Element-wise activation in float64 (machine.py:178-188); ``gelu`` (exact
    erf form, UNPINNED) is added for the ConvNeXt-style block."""
    v = np.asarray(x, dtype=F64)
    if name == "relu":
        return np.where(v > 0.0, v, 0.0)
    if name == "silu":
        return v / (1.0 + np.exp(-v))
    if name == "sigmoid":
        return 1.0 / (1.0 + np.exp(-v))
    if name == "identity":
        return v
    if name == "gelu":
        erf = np.vectorize(math.erf, otypes=[F64])
        return 0.5 * v * (1.0 + erf(v / math.sqrt(2.0)))
    raise ValueError(f"unknown activation {name!r}")


def grouped_conv2d(x, w, bias=None, stride: int = 1) -> np.ndarray:
    """Same-padded grouped cross-correlation, NHWC input, (K, R, S, T) weights,
    float64 accumulation (machine.py:191-211). Group of output channel k is
    k // (K / G). ``stride`` 2 samples the stride-1 result at even positions
    (used by the dense stem)."""
    x = np.asarray(x, dtype=F64)
    w = np.asarray(w, dtype=F64)
    n, h, wd, c = x.shape
    k, r, s, t = w.shape
    if c % t or k % (c // t):
        raise ValueError(f"group width {t} incompatible with {c} -> {k} channels")
    g = c // t
    ph, pw = r // 2, s // 2
    xp = np.zeros((n, h + 2 * ph, wd + 2 * pw, c), dtype=F64)
    xp[:, ph : ph + h, pw : pw + wd, :] = x
    xg = xp.reshape(n, h + 2 * ph, wd + 2 * pw, g, t)
    wg = w.reshape(g, k // g, r, s, t)
    acc = np.zeros((n, h, wd, g, k // g), dtype=F64)
    for dy in range(r):
        for dx in range(s):
            win = xg[:, dy : dy + h, dx : dx + wd]
            acc += np.einsum("nhwgt,gkt->nhwgk", win, wg[:, :, dy, dx, :], optimize=True)
    out = acc.reshape(n, h, wd, k)
    if bias is not None:
        out = out + np.asarray(bias, dtype=F64)
    if stride == 2:
        out = out[:, ::2, ::2, :]
    return out


def _mm(x, w, bias=None) -> np.ndarray:
    out = np.asarray(x, dtype=F64) @ np.asarray(w, dtype=F64)
    if bias is not None:
        out = out + np.asarray(bias, dtype=F64)
    return out


def layer_norm(x, gamma, beta, eps: float = 1e-6) -> np.ndarray:
    """UNPINNED. Channel LayerNorm (ConvNeXt convention: biased variance,
    eps inside the square root), float64 statistics."""
    v = np.asarray(x, dtype=F64)
    mu = v.mean(axis=-1, keepdims=True)
    var = ((v - mu) ** 2).mean(axis=-1, keepdims=True)
    return (v - mu) / np.sqrt(var + eps) * np.asarray(gamma, F64) + np.asarray(beta, F64)


# ---------------------------------------------------------------- stride 1


def ffn_block(x, u, a, v, b, activation="relu") -> np.ndarray:
    """Layer-wise FFN phi(XU + a)V + b (machine.py:228-233, schedule :339-365)."""
    y = _f32(_mm(x, u, a))
    y = _f32(phi(activation, y))
    return _f32(_mm(y, v, b))


def convnext_block(
    x,
    w_conv,
    b_conv,
    u,
    a,
    v,
    b,
    activation="relu",
    ln_gamma=None,
    ln_beta=None,
    ln_eps: float = 1e-6,
    residual: bool = True,
) -> np.ndarray:
    """The conv-first fused-block family: grouped/depthwise k x k conv + bias,
    optional channel LayerNorm, 1x1 expand + bias + phi, 1x1 project + bias,
    residual.

    With ``ln_gamma is None`` this is exactly the reference ConvFirst
    layer-wise schedule (machine.py:418-459): conv -> fp32, expand -> fp32,
    phi -> fp32, project -> fp32, + shortcut -> fp32. The LayerNorm step and
    k = 7 are UNPINNED extensions (ConvNeXt block, BASELINE config 1).
    """
    xc = _f32(grouped_conv2d(x, w_conv, b_conv))
    if ln_gamma is not None:
        xc = _f32(layer_norm(xc, ln_gamma, ln_beta, ln_eps))
    y = _f32(_mm(xc, u, a))
    y = _f32(phi(activation, y))
    z = _f32(_mm(y, v, b))
    if residual:
        z = _f32(z.astype(F64) + np.asarray(x, dtype=F32).astype(F64))
    return z


def convfirst_block(x, w_conv, b_conv, u, a, v, b, activation="relu") -> np.ndarray:
    """Reference ConvFirst, stride 1 (core.py:100-109; machine.py:418-459)."""
    return convnext_block(x, w_conv, b_conv, u, a, v, b, activation=activation)


def mbconv_block(
    x, w_exp, b_exp, w_conv, b_conv, w_sq, b_sq, w_ex, b_ex, w_prj, b_prj, activation="silu", stride: int = 1
) -> np.ndarray:
    """MBConv + squeeze-excite, layer-wise numerics (machine.py:593-646):
    expand + phi, grouped 3x3 conv + phi, SE (pool -> squeeze + ReLU ->
    excite + sigmoid -> gate), project + bias, + shortcut.

    ``stride=2`` is UNPINNED: a Triangle-3 BlurPool (stride 2, reflect pad,
    ``blurpool_2d``) follows the conv activation, SE and projection run at a
    quarter of the pixels and there is no shortcut (op-count convention of
    complexity.py:208-215)."""
    h1 = _f32(_mm(x, w_exp, b_exp))
    h1 = _f32(phi(activation, h1))
    h2 = _f32(grouped_conv2d(h1, w_conv, b_conv))
    h2 = _f32(phi(activation, h2))
    if stride == 2:
        h2 = _f32(blurpool_2d(h2))
    pool = _f32(h2.astype(F64).mean(axis=(1, 2)))
    s = _f32(_mm(pool, w_sq, b_sq))
    s = _f32(phi("relu", s))
    e = _f32(_mm(s, w_ex, b_ex))
    e = _f32(phi("sigmoid", e))
    h3 = _f32(h2.astype(F64) * e.astype(F64)[:, None, None, :])
    z = _f32(_mm(h3, w_prj, b_prj))
    if stride == 1:
        z = _f32(z.astype(F64) + np.asarray(x, dtype=F32).astype(F64))
    return z


# ------------------------------------------------------------- downsampling


def _tri(a, axis: int) -> np.ndarray:
    """UNPINNED. 1-D Triangle-3 [1, 2, 1] / 4 low-pass, stride 2, reflect pad
    of one (BlurPool, Zhang 2019). Output i reads inputs
    2i - 1, 2i, 2i + 1; index -1 reflects to 1."""
    v = np.asarray(a, dtype=F64)
    n = v.shape[axis]
    if n % 2:
        raise ValueError("blur-pool needs an even extent")
    idx = np.arange(0, n, 2)
    lo = np.abs(idx - 1)  # reflect -1 -> 1
    hi = np.minimum(idx + 1, n - 1)
    take = lambda ii: np.take(v, ii, axis=axis)  # noqa: E731
    return 0.25 * take(lo) + 0.5 * take(idx) + 0.25 * take(hi)


def blurpool_h(a) -> np.ndarray:
    return _tri(a, 1)


def blurpool_w(a) -> np.ndarray:
    return _tri(a, 2)


def blurpool_2d(a) -> np.ndarray:
    """Separable Triangle-3 x Triangle-3 / 16, stride 2 in H and W."""
    return _tri(_tri(a, 1), 2)


def convfirst_s2_block(x, w_conv, b_conv, u, a, v, b, activation="relu") -> np.ndarray:
    """UNPINNED downsampling ConvFirst. Follows the reference op-count
    convention (complexity.py:185-191: conv at HW, expand at HW/2, project at
    HW/4 -> K): grouped 3x3 conv + bias at full resolution, BlurPool along H
    (stride 2), expand + phi at (H/2, W), BlurPool along W, project + bias at
    (H/2, W/2). No shortcut."""
    xc = _f32(grouped_conv2d(x, w_conv, b_conv))
    xc = _f32(blurpool_h(xc))
    y = _f32(_mm(xc, u, a))
    y = _f32(phi(activation, y))
    y = _f32(blurpool_w(y))
    return _f32(_mm(y, v, b))


# --------------------------------------------------------------- stem, head


def stem_block(x, w, b, activation="relu") -> np.ndarray:
    """UNPINNED. Dense 3x3 stride-2 conv (pad 1) + bias + phi
    (core.py:135-141; ops complexity.py:147-151)."""
    return _f32(phi(activation, _f32(grouped_conv2d(x, w, b, stride=2))))


def head_block(x, w1, b1, w2, b2, activation="relu") -> np.ndarray:
    """UNPINNED. 1x1 conv to the embedding + bias + phi, global average pool,
    linear classifier (core.py:144-152; ops complexity.py:153-157)."""
    h = _f32(phi(activation, _f32(_mm(x, w1, b1))))
    pool = _f32(h.astype(F64).mean(axis=(1, 2)))
    return _f32(_mm(pool, w2, b2))


# ------------------------------------------------- ConvNeXt-T units (UNPINNED)


def patch_stem_block(x, w, b, gamma, beta, eps: float = 1e-6) -> np.ndarray:
    """UNPINNED (ConvNeXt-T, no reference constructor). p x p
    stride-p conv (w: (k, p, p, c)) + bias, then channel LayerNorm."""
    x = np.asarray(x, dtype=F64)
    n, hh, ww, c = x.shape
    k, p = w.shape[0], w.shape[1]
    pt = x.reshape(n, hh // p, p, ww // p, p, c).transpose(0, 1, 3, 2, 4, 5).reshape(n, hh // p, ww // p, p * p * c)
    y = _f32(pt @ np.asarray(w, dtype=F64).reshape(k, -1).T + np.asarray(b, dtype=F64))
    return _f32(layer_norm(y, gamma, beta, eps))


def downsample_block(x, gamma, beta, w, b, eps: float = 1e-6) -> np.ndarray:
    """UNPINNED (ConvNeXt-T). Channel LayerNorm, then 2x2 stride-2 conv
    (w: (k, 2, 2, c)) + bias."""
    xn = _f32(layer_norm(x, gamma, beta, eps)).astype(F64)
    n, hh, ww, c = xn.shape
    k = w.shape[0]
    pt = xn.reshape(n, hh // 2, 2, ww // 2, 2, c).transpose(0, 1, 3, 2, 4, 5).reshape(n, hh // 2, ww // 2, 4 * c)
    return _f32(pt @ np.asarray(w, dtype=F64).reshape(k, -1).T + np.asarray(b, dtype=F64))


def ln_head_block(x, gamma, beta, w, b, eps: float = 1e-6) -> np.ndarray:
    """UNPINNED (ConvNeXt-T). Global average pool, channel LayerNorm, linear
    classifier (w: (c, classes))."""
    pool = _f32(np.asarray(x, dtype=F64).mean(axis=(1, 2)))
    f = _f32(layer_norm(pool, gamma, beta, eps))
    return _f32(_mm(f, w, b))
