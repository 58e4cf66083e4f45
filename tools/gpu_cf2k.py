"""cf2 parity sweep over output widths (debug helper)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from oracle import model as om
from paper_2404_03617_b200.blocks import init_weights
from paper_2404_03617_b200.core import ConvFirst, MBConv, TensorDims
from paper_2404_03617_b200.machine import build_schedule, execute_numeric

def run(block, dims, k):
    rng = np.random.default_rng(0)
    s = build_schedule(block, dims, out_channels=k)
    w = {n: v.astype(np.float16).astype(np.float32) for n, v in init_weights(s, rng).items()}
    x = rng.standard_normal((dims.n, dims.h, dims.w, dims.c)).astype(np.float16).astype(np.float32)
    got = execute_numeric(s, dict(w, x=x))
    ref = om.unit_forward(block, w, x)
    err = np.abs(got - ref).max() / np.abs(ref).max()
    bad = np.abs(got - ref).max(axis=(0, 1, 2)) / np.abs(ref).max()
    print(type(block).__name__, dims, k, f"max_rel {err:.3g}", "bad channels", np.nonzero(bad > 1e-2)[0][:20].tolist(), flush=True)

for c, k, hw in [(48, 64, 56), (48, 80, 56), (48, 96, 56), (48, 112, 56), (48, 80, 28), (32, 80, 56), (64, 80, 28)]:
    run(ConvFirst(8, 6, 2), TensorDims(2, hw, hw, c), k)
