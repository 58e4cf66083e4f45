"""The tcgen05 GEMM (wl_gemm, csrc/gemm.cu) against a plain PyTorch fp32
reference of the same op: D = act(A B^T + bias) (+ res), fp16 storage, fp32
accumulation. Tolerance: max|d - ref| / max|ref| <= 1e-2 (fp16 output rounding
and the half-precision tanh-form GELU)."""

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2404_03617_b200 import _lib  # noqa: E402


def _ref(a, b, bias, act, res):
    y = a.float() @ b.float().T
    if bias is not None:
        y = y + bias
    if act == "gelu":
        y = torch.nn.functional.gelu(y)
    elif act == "relu":
        y = torch.relu(y)
    elif act == "silu":
        y = torch.nn.functional.silu(y)
    if res is not None:
        y = y + res.float()
    return y


@pytest.mark.parametrize("m,k,n,act,bias,res", [
    (1, 8, 8, "identity", False, False),          # smallest legal shape
    (300, 48, 96, "identity", True, False),       # K < 64 (TMA zero fill), N < 128
    (1000, 192, 768, "gelu", True, False),        # M tail, N = 3 x 256
    (513, 768, 192, "identity", True, True),      # residual through the staging tile
    (130, 1280, 1000, "identity", True, False),   # the classifier shape, N tail (1000 = 3 x 256 + 232)
    (257, 384, 1536, "silu", True, False),
    (64, 96, 384, "relu", False, True),
])
def test_gemm_vs_torch(m, k, n, act, bias, res):
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n)
    a = torch.randn(m, k, device="cuda", generator=g).half()
    b = (torch.randn(n, k, device="cuda", generator=g) / k ** 0.5).half()
    bi = torch.randn(n, device="cuda", generator=g) if bias else None
    r = torch.randn(m, n, device="cuda", generator=g).half() if res else None
    _lib.lib().wl_init(0)
    out = _lib.gemm(a, b, bi, act, r)
    torch.cuda.synchronize()
    ref = _ref(a, b, bi, act, r)
    err = (out.float() - ref).abs().max().item() / max(ref.abs().max().item(), 1e-6)
    assert torch.isfinite(out.float()).all() and err <= 1e-2, err


def test_gemm_rejects_bad_strides():
    a = torch.zeros(16, 20, device="cuda").half()  # K = 20: rows are not 16-byte multiples
    b = torch.zeros(16, 20, device="cuda").half()
    with pytest.raises(ValueError):
        _lib.gemm(a, b)


def test_gemm_bf16_vs_torch():
    g = torch.Generator(device="cuda").manual_seed(3)
    a = torch.randn(700, 384, device="cuda", generator=g).bfloat16()
    b = (torch.randn(1536, 384, device="cuda", generator=g) / 384 ** 0.5).bfloat16()
    bias = torch.randn(1536, device="cuda", generator=g)
    r = torch.randn(700, 1536, device="cuda", generator=g).bfloat16()
    out = _lib.gemm(a, b, bias, "gelu", r)
    torch.cuda.synchronize()
    ref = _ref(a, b, bias, "gelu", r)
    assert out.dtype == torch.bfloat16
    err = (out.float() - ref).abs().max().item() / ref.abs().max().item()
    assert err <= 4e-2, err
