"""GPU parity of the ConvNeXt-T units (BASELINE config 4) and the FFN block,
through the C ABI, against the CPU oracle (oracle/blocks.py; its ConvNeXt
pieces are pinned to torch.nn.functional in tests/test_oracle_torch.py).
Tolerance as tests/test_gpu_parity.py (fp16 storage, fp32 accumulation):
max-rel 1e-2, L2-rel 2e-3 per unit; logits 2e-2 / 1e-2."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import model as om  # noqa: E402
from paper_2404_03617_b200.blocks import FusedBlock, init_weights  # noqa: E402
from paper_2404_03617_b200.convnext import ConvNeXtSpec, convnext_tiny  # noqa: E402
from paper_2404_03617_b200.core import FFN, ConvNeXtBlock, Downsample, LNHead, PatchifyStem, TensorDims  # noqa: E402
from paper_2404_03617_b200.machine import build_schedule, execute_numeric  # noqa: E402
from paper_2404_03617_b200.scheduler import FusedNetwork  # noqa: E402

from test_gpu_parity import close, r16  # noqa: E402


def _case(block, dims, k=None, seed=0):
    rng = np.random.default_rng(seed)
    s = build_schedule(block, dims, out_channels=k)
    w = {n: v.astype(np.float16).astype(np.float32) for n, v in init_weights(s, rng).items()}
    x = r16(rng, s.tensor("x").dims)
    return s, w, x


CASES = [
    # FFN rows (tcgen05 GEMM pair): M tails, N = 96 / 192-tiles / 256-tiles, K tails (48 -> 64)
    ("ffn_c96", FFN(4, "gelu"), TensorDims(1, 10, 100, 96), None),
    ("ffn_c48_relu", FFN(4, "relu"), TensorDims(1, 7, 9, 48), None),
    ("ffn_c192_silu", FFN(4, "silu"), TensorDims(2, 5, 33, 192), None),
    ("ffn_c768", FFN(4, "gelu"), TensorDims(1, 1, 200, 768), None),
    # the fused kernel (hidden on chip, ffn.cu): HC = 128 (C <= 256) / 64 (C = 384), multi-tile grids
    ("ffn_fused_c384", FFN(4, "gelu"), TensorDims(2, 14, 14, 384), None),
    ("ffn_fused_c256_identity", FFN(2, "identity"), TensorDims(1, 3, 700, 256), None),
    ("ffn_fused_c128_many_tiles", FFN(4, "relu"), TensorDims(4, 56, 100, 128), None),
    # ConvNeXt-T units at their network shapes (small batch)
    ("patch_stem_224", PatchifyStem(96), TensorDims(2, 224, 224, 3), None),
    ("patch_stem_rect", PatchifyStem(64, 4), TensorDims(1, 40, 24, 3), None),
    ("downsample_96_192", Downsample(192), TensorDims(2, 56, 56, 96), None),
    ("downsample_384_768", Downsample(768), TensorDims(2, 14, 14, 384), None),
    ("ln_head_768", LNHead(1000), TensorDims(3, 7, 7, 768), None),
    ("ln_head_batch_over_128", LNHead(1000), TensorDims(130, 7, 7, 768), None),
    ("convnext_wide_192", ConvNeXtBlock(7, 4, "gelu"), TensorDims(2, 28, 28, 192), None),
    ("convnext_wide_384", ConvNeXtBlock(7, 4, "gelu"), TensorDims(2, 14, 14, 384), None),
    ("convnext_wide_768", ConvNeXtBlock(7, 4, "gelu"), TensorDims(2, 7, 7, 768), None),
    ("convnext_wide_rect_256", ConvNeXtBlock(7, 4, "gelu"), TensorDims(1, 9, 13, 256), None),
    ("convnext_wide_3x3", ConvNeXtBlock(3, 4, "gelu"), TensorDims(1, 12, 12, 192), None),
]


@pytest.mark.parametrize("name,block,dims,k", CASES, ids=[c[0] for c in CASES])
def test_unit_vs_oracle(name, block, dims, k):
    s, w, x = _case(block, dims, k)
    got = execute_numeric(s, dict(w, x=x))
    close(got, om.unit_forward(block, w, x))


def test_convnext_tiny_per_unit_and_logits():
    spec = convnext_tiny(224)
    m = FusedNetwork(spec, batch=2, seed=21)
    rng = np.random.default_rng(2)
    x = r16(rng, (2, 224, 224, 3))
    out = m(torch.from_numpy(x).half().cuda())
    torch.cuda.synchronize()
    src = x
    for u, inst in zip(m.units, m.instances):
        got = u.out.float().cpu().numpy()
        ref = om.unit_forward(inst.block, u.module.weights, src)
        close(got.reshape(ref.shape), ref)
        src = got.reshape(ref.shape)
    ref = om.network_forward(m.instances, m.weights(), x)
    close(out.float().cpu().numpy(), ref, max_rel=2e-2, l2_rel=1e-2)


def test_convnext_tiny_b128_sampled_images():
    """BASELINE config 4 at full size: images 0, 63, 127 of the b128 forward
    match the oracle unit by unit (hidden row batches of the wide blocks and
    the multi-tile GEMM grids all in play)."""
    m = FusedNetwork(convnext_tiny(224), batch=128, seed=5)
    m.x.normal_()
    m.replay()
    torch.cuda.synchronize()
    pick = [0, 63, 127]
    src = m.x.float().cpu().numpy()[pick]
    for u, inst in zip(m.units, m.instances):
        got = u.out.float().cpu().numpy()[pick]
        ref = om.unit_forward(inst.block, u.module.weights, src)
        close(got.reshape(ref.shape), ref)
        src = got.reshape(ref.shape)


def test_convnext_graph_equals_eager():
    spec = ConvNeXtSpec("mini", (64, 64), depths=(1, 1, 2, 1), dims=(96, 192, 384, 768), num_classes=1000)
    m = FusedNetwork(spec, batch=3, seed=1)
    m.x.normal_()
    m.launch_all()
    eager = m.output.clone()
    m.capture()
    m.replay()
    torch.cuda.synchronize()
    assert torch.equal(eager, m.output)


def test_ffn_module_device_path():
    s, w, x = _case(FFN(4, "gelu"), TensorDims(2, 14, 14, 384))
    mod = FusedBlock(s.block, s.dims, weights=w)
    dev = mod.launch  # raw launch through the C ABI on the current stream
    xd = torch.from_numpy(x).half().cuda()
    out = torch.empty(mod.out_shape, dtype=torch.float16, device="cuda")
    dev(xd, out)
    torch.cuda.synchronize()
    close(out.float().cpu().numpy(), om.unit_forward(s.block, w, x))


# ---------------------------------------------------------------- bf16
BF_MAX, BF_L2 = 4e-2, 8e-3  # bf16 storage (8-bit mantissa), fp32 accumulation


def _bf16(a):
    return torch.from_numpy(np.asarray(a, np.float32)).bfloat16().float().numpy()


@pytest.mark.parametrize("name,block,dims", [
    ("ffn_c96", FFN(4, "gelu"), TensorDims(1, 10, 100, 96)),
    ("ffn_c384", FFN(4, "gelu"), TensorDims(2, 14, 14, 384)),
    ("patch_stem", PatchifyStem(96), TensorDims(2, 64, 64, 3)),
    ("downsample", Downsample(192), TensorDims(2, 28, 28, 96)),
    ("ln_head", LNHead(1000), TensorDims(3, 7, 7, 768)),
    ("convnext_96", ConvNeXtBlock(7, 4, "gelu"), TensorDims(2, 28, 28, 96)),
    ("convnext_384", ConvNeXtBlock(7, 4, "gelu"), TensorDims(2, 14, 14, 384)),
    ("convnext_768", ConvNeXtBlock(7, 4, "gelu"), TensorDims(2, 7, 7, 768)),
])
def test_bf16_units_vs_oracle(name, block, dims):
    s, w, x = _case(block, dims)
    w = {k: _bf16(v) for k, v in w.items()}
    x = _bf16(x)
    m = FusedBlock(s.block, s.dims, weights=w, dtype=torch.bfloat16)
    xd = torch.from_numpy(x).cuda().bfloat16().reshape(m.in_shape if block.kind != "ffn" else x.shape)
    out = torch.empty(m.out_shape, dtype=torch.bfloat16, device="cuda")
    m.launch(xd, out)
    torch.cuda.synchronize()
    close(out.float().cpu().numpy(), om.unit_forward(block, w, x), max_rel=BF_MAX, l2_rel=BF_L2)


def test_convnext_tiny_bf16_logits():
    """ConvNeXt-T end to end in bf16 storage."""
    m = FusedNetwork(convnext_tiny(224), batch=2, seed=21, dtype=torch.bfloat16)
    rng = np.random.default_rng(2)
    x = _bf16(rng.standard_normal((2, 224, 224, 3)))
    out = m(torch.from_numpy(x).cuda().bfloat16())
    torch.cuda.synchronize()
    src = x
    for u, inst in zip(m.units, m.instances):
        got = u.out.float().cpu().numpy()
        ref = om.unit_forward(inst.block, {k: _bf16(v) for k, v in u.module.weights.items()}, src)
        close(got.reshape(ref.shape), ref, max_rel=BF_MAX, l2_rel=BF_L2)
        src = got.reshape(ref.shape)
    assert out.dtype == torch.bfloat16 and torch.isfinite(out.float()).all()


def test_fp16_only_families_refuse_bf16():
    from paper_2404_03617_b200.core import MBConv

    with pytest.raises(Exception):
        FusedBlock(MBConv(8, 4, 0.25), TensorDims(1, 14, 14, 128), dtype=torch.bfloat16)
