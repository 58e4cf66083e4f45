"""The reference's LAYER_WISE schedules on the device (layerwise.cu: one
launch per layer, every intermediate through HBM) against the reference's
own layer-wise golden outputs, the CPU oracle, and the fused kernels on the
same inputs. Tolerance as tests/test_gpu_parity.py (fp16 storage, fp32
accumulation: max-rel 1e-2, L2-rel 2e-3)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import model as om  # noqa: E402
from oracle.fixtures import golden_names, load_golden  # noqa: E402
from paper_2404_03617_b200.blocks import FusedBlock, init_weights  # noqa: E402
from paper_2404_03617_b200.core import FFN, ConvFirst, ExecutionScheme, MBConv, TensorDims  # noqa: E402
from paper_2404_03617_b200.machine import build_schedule, execute_numeric  # noqa: E402

from test_gpu_parity import close, r16  # noqa: E402

LW = ExecutionScheme.LAYER_WISE


@pytest.mark.parametrize("name", golden_names())
def test_layer_wise_golden_vectors(name):
    meta, ins, out_lw, _ = load_golden(name)
    kinds = {"ConvFirst": ConvFirst, "MBConv": MBConv, "FFN": FFN}
    s = build_schedule(kinds[meta["block"]](**meta["params"]), TensorDims(*meta["dims"]), LW)
    close(execute_numeric(s, ins), out_lw)


CASES = [
    ("cf_pico", ConvFirst(8, 3), TensorDims(2, 112, 112, 16)),
    ("cf_c1", ConvFirst(8, 6), TensorDims(2, 56, 56, 96)),
    ("cf_silu", ConvFirst(8, 4, 1, "silu"), TensorDims(3, 28, 28, 64)),
    ("cf_dw", ConvFirst(1, 4, 1, "gelu"), TensorDims(2, 28, 28, 48)),
    ("mb_14", MBConv(8, 4, 0.25), TensorDims(4, 14, 14, 128)),
    ("mb_7", MBConv(8, 4, 0.25), TensorDims(4, 7, 7, 256)),
    ("mb_dw", MBConv(1, 4, 0.25), TensorDims(2, 28, 28, 80)),
    ("mb_big_hidden", MBConv(8, 6, 0.25), TensorDims(2, 14, 14, 256)),  # 1536 hidden channels: 24 conv slices, 55 KB SE partials
    ("ffn", FFN(4, "gelu"), TensorDims(2, 14, 14, 96)),
]


@pytest.mark.parametrize("name,block,dims", CASES, ids=[c[0] for c in CASES])
def test_layer_wise_matches_oracle_and_fused(name, block, dims):
    rng = np.random.default_rng(5)
    s = build_schedule(block, dims, LW)
    w = {n: v.astype(np.float16).astype(np.float32) for n, v in init_weights(s, rng).items()}
    x = r16(rng, next(t.dims for t in s.tensors if t.name == "x"))
    lw = execute_numeric(s, dict(w, x=x))
    close(lw, om.unit_forward(block, w, x))
    fused = execute_numeric(build_schedule(block, dims), dict(w, x=x))
    close(lw, fused)


def test_layer_wise_block_module_graph_equals_eager():
    dims = TensorDims(8, 14, 14, 128)
    blk = FusedBlock(MBConv(8, 4, 0.25), dims, seed=3, scheme=LW)
    x = torch.randn(dims.n, dims.h, dims.w, dims.c, device="cuda").half()
    eager = blk(x)
    out = torch.empty_like(eager)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        blk.launch(x, out)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        blk.launch(x, out)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager)
    fused = FusedBlock(MBConv(8, 4, 0.25), dims, weights=blk.weights)
    close(eager.float().cpu().numpy(), fused(x).float().cpu().numpy())


@pytest.mark.parametrize("argv", [
    ["--block", "convfirst", "--channels", "32", "--expansion", "6", "--size", "28x28", "--batch", "2", "--time", "5"],
    ["--block", "mbconv", "--channels", "128", "--size", "14x14", "--batch", "4", "--time", "5"],
    ["--block", "ffn", "--channels", "96", "--size", "7x7", "--batch", "2"],
])
def test_simulate_b200_fused_vs_layer_wise(argv, capsys):
    """The reference's simulate check with both schedules on the device."""
    from paper_2404_03617_b200 import simulate

    assert simulate.main(argv) == simulate.EXIT_OK
    out = capsys.readouterr().out
    assert "layerwise" in out and "blockfusion" in out and "relative error" in out
