"""The CPU oracle against the reference's own outputs (golden vectors made by
tests/golden/make_golden.py from the unmodified reference execute_numeric)
and against the SPEC known-answer cases."""

import numpy as np
import pytest

import oracle
from oracle.fixtures import golden_names, load_golden

CF_ORDER = ["x", "w_conv", "b_conv", "u", "a", "v", "b"]
MB_ORDER = ["x", "w_exp", "b_exp", "w_conv", "b_conv", "w_sq", "b_sq", "w_ex", "b_ex", "w_prj", "b_prj"]


@pytest.mark.parametrize("name", golden_names())
def test_oracle_matches_reference_layerwise(name):
    meta, ins, out_lw, out_bf = load_golden(name)
    act = meta["params"]["activation"]
    if meta["block"] == "ConvFirst":
        got = oracle.convfirst_block(*[ins[k] for k in CF_ORDER], activation=act)
    elif meta["block"] == "MBConv":
        got = oracle.mbconv_block(*[ins[k] for k in MB_ORDER], activation=act)
    else:
        x = ins["x"]
        got = oracle.ffn_block(x, ins["u"], ins["a"], ins["v"], ins["b"], activation=act)
    scale = np.abs(out_lw).max()
    # same float32 storage points, float64 accumulation: equal up to BLAS summation order
    assert np.abs(got - out_lw).max() <= 2e-6 * scale
    # and the reference's own fused schedule agrees with its layer-wise one
    assert np.abs(out_bf - out_lw).max() <= 1e-4 * scale


def test_ffn_hand_case():
    # SPEC known answer: X = [[1]], U = [[2]], a = [1], V = [[3]], b = [-1] -> relu(3) * 3 - 1 = 8
    got = oracle.ffn_block(np.array([[1.0]]), np.array([[2.0]]), np.array([1.0]), np.array([[3.0]]), np.array([-1.0]))
    assert got.tolist() == [[8.0]]


def test_zero_input_zero_weights_gives_zero():
    x = np.zeros((1, 6, 6, 16), np.float32)
    z = oracle.convfirst_block(x, np.zeros((16, 3, 3, 8)), np.zeros(16), np.zeros((16, 48)), np.zeros(48),
                               np.zeros((48, 16)), np.zeros(16))
    assert not z.any()


def test_convnext_without_norm_is_convfirst():
    rng = np.random.default_rng(3)
    x = rng.standard_normal((1, 8, 8, 16)).astype(np.float32)
    w = rng.standard_normal((16, 3, 3, 1)).astype(np.float32)
    args = [rng.standard_normal(s).astype(np.float32) for s in ((16,), (16, 64), (64,), (64, 16), (16,))]
    a = oracle.convnext_block(x, w, *args, activation="relu")
    b = oracle.convfirst_block(x, w, *args)
    assert np.array_equal(a, b)


def test_layer_norm_statistics():
    rng = np.random.default_rng(4)
    x = rng.standard_normal((2, 3, 3, 32)) * 5 + 2
    y = oracle.layer_norm(x, np.ones(32), np.zeros(32))
    assert np.allclose(y.mean(-1), 0, atol=1e-9) and np.allclose(y.var(-1), 1, atol=1e-4)


def test_blurpool_reflect_and_constant():
    a = np.ones((1, 4, 6, 2))
    assert np.allclose(oracle.blurpool_2d(a), 1.0)  # low-pass preserves constants
    r = np.arange(8, dtype=float).reshape(1, 8, 1, 1)
    out = oracle.blurpool_h(r)[0, :, 0, 0]
    # output 0 reads rows (-1 -> 1), 0, 1
    assert out[0] == pytest.approx(0.25 * 1 + 0.5 * 0 + 0.25 * 1)
    assert out[1] == pytest.approx(0.25 * 1 + 0.5 * 2 + 0.25 * 3)


def test_stem_is_strided_dense_conv():
    rng = np.random.default_rng(5)
    x = rng.standard_normal((1, 6, 6, 3)).astype(np.float32)
    w = rng.standard_normal((4, 3, 3, 3)).astype(np.float32)
    b = np.zeros(4, np.float32)
    z = oracle.stem_block(x, w, b, activation="identity")
    xp = np.pad(x, ((0, 0), (1, 1), (1, 1), (0, 0)))
    manual = np.einsum("ijc,kijc->k", xp[0, 2:5, 2:5, :], w)
    assert np.allclose(z[0, 1, 1], manual, rtol=1e-5, atol=1e-5)
