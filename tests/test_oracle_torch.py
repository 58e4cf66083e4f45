"""Pins the oracle pieces the reference cannot execute (stem, stride-2
BlurPool blocks, LayerNorm, GELU, 7x7 depthwise, head; oracle/blocks.py)
against independent published implementations: torch.nn.functional in
float64 on the CPU. The oracle's own float32 storage points are kept, so the
comparison is to float32 rounding."""

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
F = torch.nn.functional

TOL = 2e-6  # relative to max|ref|: float32 storage in the oracle vs float64 torch


def t64(a):
    return torch.from_numpy(np.asarray(a, dtype=np.float64))


def nchw(x):
    return t64(x).permute(0, 3, 1, 2)


def nhwc(t):
    return t.permute(0, 2, 3, 1).numpy()


def close(got, ref, tol=TOL):
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    assert got.shape == ref.shape
    assert np.abs(got - ref).max() <= tol * max(np.abs(ref).max(), 1e-12)


def conv_weight(w):
    """(K, R, S, T) reference layout -> torch (K, T, R, S)."""
    return t64(w).permute(0, 3, 1, 2)


def blur_torch(x_nchw):
    """BlurPool (Zhang 2019): reflect pad 1, depthwise [1,2,1] x [1,2,1] / 16, stride 2."""
    c = x_nchw.shape[1]
    k1 = torch.tensor([1.0, 2.0, 1.0], dtype=torch.float64)
    k = (k1[:, None] * k1[None, :] / 16.0).expand(c, 1, 3, 3).contiguous()
    return F.conv2d(F.pad(x_nchw, (1, 1, 1, 1), mode="reflect"), k, stride=2, groups=c)


@pytest.fixture
def rng():
    return np.random.default_rng(2024)


@pytest.mark.parametrize("t,k", [(8, 3), (1, 3), (1, 7), (4, 5)])
def test_grouped_conv_vs_torch(rng, t, k):
    x = rng.standard_normal((2, 11, 9, 32))
    w = rng.standard_normal((32, k, k, t))
    b = rng.standard_normal(32)
    got = oracle.grouped_conv2d(x, w, b)
    ref = F.conv2d(nchw(x), conv_weight(w), t64(b), padding=k // 2, groups=32 // t)
    close(got, nhwc(ref), 1e-12)


def test_stem_vs_torch(rng):
    x = rng.standard_normal((2, 18, 14, 3)).astype(np.float32)
    w = rng.standard_normal((16, 3, 3, 3)).astype(np.float32)
    b = rng.standard_normal(16).astype(np.float32)
    got = oracle.stem_block(x, w, b)
    ref = F.relu(F.conv2d(nchw(x), conv_weight(w), t64(b), stride=2, padding=1))
    close(got, nhwc(ref))


def test_layer_norm_vs_torch(rng):
    x = rng.standard_normal((2, 5, 5, 96)) * 3 + 7  # large mean: the statistic is two-pass
    g, bta = rng.standard_normal(96), rng.standard_normal(96)
    got = oracle.layer_norm(x, g, bta, 1e-6)
    ref = F.layer_norm(t64(x), (96,), t64(g), t64(bta), eps=1e-6)
    close(got, ref.numpy(), 1e-12)


@pytest.mark.parametrize("act,fn", [("gelu", lambda v: F.gelu(v)), ("silu", F.silu), ("relu", F.relu),
                                    ("sigmoid", torch.sigmoid)])
def test_activations_vs_torch(rng, act, fn):
    v = rng.standard_normal(4096) * 4
    close(oracle.phi(act, v), fn(t64(v)).numpy(), 1e-12)


def test_blurpool_vs_reflect_padded_depthwise_conv(rng):
    x = rng.standard_normal((2, 12, 10, 8))
    close(oracle.blurpool_2d(x), nhwc(blur_torch(nchw(x))), 1e-12)


def test_convnext_block_vs_torch(rng):
    c, hid = 32, 128
    x = rng.standard_normal((2, 9, 9, c)).astype(np.float32)
    w = (rng.standard_normal((c, 7, 7, 1)) * 0.2).astype(np.float32)
    bc, g, bt = (rng.standard_normal(c).astype(np.float32) for _ in range(3))
    u = (rng.standard_normal((c, hid)) * 0.2).astype(np.float32)
    a = rng.standard_normal(hid).astype(np.float32)
    v = (rng.standard_normal((hid, c)) * 0.1).astype(np.float32)
    b = rng.standard_normal(c).astype(np.float32)
    got = oracle.convnext_block(x, w, bc, u, a, v, b, activation="gelu", ln_gamma=g, ln_beta=bt)
    h = F.conv2d(nchw(x), conv_weight(w), t64(bc), padding=3, groups=c).permute(0, 2, 3, 1)
    h = F.layer_norm(h, (c,), t64(g), t64(bt), eps=1e-6)
    h = F.gelu(h @ t64(u) + t64(a)) @ t64(v) + t64(b)
    close(got, (h + t64(x)).numpy(), 1e-5)


def test_convfirst_stride2_vs_torch(rng):
    """conv@HW -> blur_H -> expand@(H/2,W) -> phi -> blur_W -> project (oracle
    convention, complexity.py:185-191) equals, by linearity of the blur along
    W, torch's conv -> BlurPool-H -> expand -> phi -> BlurPool-W -> project."""
    c, hid, k = 16, 96, 32
    x = rng.standard_normal((2, 12, 10, c)).astype(np.float32)
    w = (rng.standard_normal((c, 3, 3, 8)) * 0.3).astype(np.float32)
    bc = rng.standard_normal(c).astype(np.float32)
    u = (rng.standard_normal((c, hid)) * 0.3).astype(np.float32)
    a = rng.standard_normal(hid).astype(np.float32)
    v = (rng.standard_normal((hid, k)) * 0.1).astype(np.float32)
    b = rng.standard_normal(k).astype(np.float32)
    got = oracle.convfirst_s2_block(x, w, bc, u, a, v, b)
    h = F.conv2d(nchw(x), conv_weight(w), t64(bc), padding=1, groups=c // 8)
    k1 = torch.tensor([0.25, 0.5, 0.25], dtype=torch.float64)
    bh = k1.view(1, 1, 3, 1).expand(c, 1, 3, 1).contiguous()
    h = F.conv2d(F.pad(h, (0, 0, 1, 1), mode="reflect"), bh, stride=(2, 1), groups=c)
    y = F.relu(h.permute(0, 2, 3, 1) @ t64(u) + t64(a)).permute(0, 3, 1, 2)
    bw = k1.view(1, 1, 1, 3).expand(hid, 1, 1, 3).contiguous()
    y = F.conv2d(F.pad(y, (1, 1, 0, 0), mode="reflect"), bw, stride=(1, 2), groups=hid)
    z = y.permute(0, 2, 3, 1) @ t64(v) + t64(b)
    close(got, z.numpy(), 1e-5)


def test_mbconv_stride2_vs_torch(rng):
    c, hid, sq, k = 16, 64, 4, 32
    x = rng.standard_normal((2, 10, 12, c)).astype(np.float32)
    we = (rng.standard_normal((c, hid)) * 0.3).astype(np.float32)
    be = rng.standard_normal(hid).astype(np.float32)
    wc = (rng.standard_normal((hid, 3, 3, 8)) * 0.3).astype(np.float32)
    bc = rng.standard_normal(hid).astype(np.float32)
    wsq = (rng.standard_normal((hid, sq)) * 0.3).astype(np.float32)
    bsq = rng.standard_normal(sq).astype(np.float32)
    wex = (rng.standard_normal((sq, hid)) * 0.3).astype(np.float32)
    bex = rng.standard_normal(hid).astype(np.float32)
    wp = (rng.standard_normal((hid, k)) * 0.1).astype(np.float32)
    bp = rng.standard_normal(k).astype(np.float32)
    got = oracle.mbconv_block(x, we, be, wc, bc, wsq, bsq, wex, bex, wp, bp, activation="silu", stride=2)
    h1 = F.silu(t64(x) @ t64(we) + t64(be)).permute(0, 3, 1, 2)
    h2 = F.silu(F.conv2d(h1, conv_weight(wc), t64(bc), padding=1, groups=hid // 8))
    h2 = blur_torch(h2)
    e = torch.sigmoid(F.relu(F.adaptive_avg_pool2d(h2, 1).flatten(1) @ t64(wsq) + t64(bsq)) @ t64(wex) + t64(bex))
    z = (h2 * e[:, :, None, None]).permute(0, 2, 3, 1) @ t64(wp) + t64(bp)
    close(got, z.numpy(), 1e-5)


def test_head_vs_torch(rng):
    x = rng.standard_normal((3, 7, 7, 32)).astype(np.float32)
    w1 = (rng.standard_normal((32, 64)) * 0.2).astype(np.float32)
    b1 = rng.standard_normal(64).astype(np.float32)
    w2 = (rng.standard_normal((64, 10)) * 0.2).astype(np.float32)
    b2 = rng.standard_normal(10).astype(np.float32)
    got = oracle.head_block(x, w1, b1, w2, b2)
    e = F.relu(F.conv2d(nchw(x), t64(w1).T[:, :, None, None], t64(b1)))
    ref = F.linear(F.adaptive_avg_pool2d(e, 1).flatten(1), t64(w2).T, t64(b2))
    close(got, ref.numpy())


# ------------------------------------------------- ConvNeXt-T units (UNPINNED)


def test_patch_stem_vs_torch(rng):
    x = rng.standard_normal((2, 16, 12, 3))
    w = rng.standard_normal((32, 4, 4, 3))
    b, g, be = rng.standard_normal(32), 1 + 0.1 * rng.standard_normal(32), 0.1 * rng.standard_normal(32)
    got = oracle.patch_stem_block(x, w, b, g, be)
    y = F.conv2d(nchw(x), conv_weight(w), t64(b), stride=4).permute(0, 2, 3, 1)
    ref = F.layer_norm(y, (32,), t64(g), t64(be), eps=1e-6).numpy()
    close(got, ref)


def test_downsample_vs_torch(rng):
    x = rng.standard_normal((2, 8, 6, 24))
    w = rng.standard_normal((48, 2, 2, 24))
    b, g, be = rng.standard_normal(48), 1 + 0.1 * rng.standard_normal(24), 0.1 * rng.standard_normal(24)
    got = oracle.downsample_block(x, g, be, w, b)
    xn = F.layer_norm(t64(x), (24,), t64(g), t64(be), eps=1e-6).permute(0, 3, 1, 2)
    ref = nhwc(F.conv2d(xn, conv_weight(w), t64(b), stride=2))
    close(got, ref)


def test_ln_head_vs_torch(rng):
    x = rng.standard_normal((3, 7, 7, 64))
    w, b = rng.standard_normal((64, 40)), rng.standard_normal(40)
    g, be = 1 + 0.1 * rng.standard_normal(64), 0.1 * rng.standard_normal(64)
    got = oracle.ln_head_block(x, g, be, w, b)
    f = F.layer_norm(t64(x).mean(dim=(1, 2)), (64,), t64(g), t64(be), eps=1e-6)
    ref = F.linear(f, t64(w).T, t64(b)).numpy()
    close(got, ref)


def test_convnext_block_vs_torch_module(rng):
    """The ConvNeXt block as the original code writes it (dwconv groups=C ->
    permute -> LayerNorm -> Linear -> GELU(erf) -> Linear -> + x)."""
    c = 48
    x = rng.standard_normal((2, 9, 10, c))
    wdw, bdw = rng.standard_normal((c, 7, 7, 1)) / 7, rng.standard_normal(c)
    g, be = 1 + 0.1 * rng.standard_normal(c), 0.1 * rng.standard_normal(c)
    u, a = rng.standard_normal((c, 4 * c)) / np.sqrt(c), rng.standard_normal(4 * c)
    v, b = rng.standard_normal((4 * c, c)) / np.sqrt(4 * c), rng.standard_normal(c)
    got = oracle.convnext_block(x, wdw, bdw, u, a, v, b, activation="gelu", ln_gamma=g, ln_beta=be)
    y = F.conv2d(nchw(x), conv_weight(wdw), t64(bdw), padding=3, groups=c).permute(0, 2, 3, 1)
    y = F.layer_norm(y, (c,), t64(g), t64(be), eps=1e-6)
    y = F.linear(F.gelu(F.linear(y, t64(u).T, t64(a))), t64(v).T, t64(b))
    close(got, (y + t64(x)).numpy(), tol=1e-5)
