"""Run one fused block (or a list) a few times for ncu."""
import sys, os, argparse
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_03617_b200.core import ConvFirst, MBConv, Stem, Head, ConvNeXtBlock, TensorDims, FFN, PatchifyStem, Downsample, LNHead
from paper_2404_03617_b200.blocks import FusedBlock

CASES = {
    "mb14": (MBConv(8, 4, 0.25), TensorDims(128, 14, 14, 128), None),
    "mb7": (MBConv(8, 4, 0.25), TensorDims(128, 7, 7, 128), None),
    "mbs2_28": (MBConv(8, 4, 0.25, 2), TensorDims(128, 28, 28, 48), 128),
    "mbs2_14": (MBConv(8, 4, 0.25, 2), TensorDims(128, 14, 14, 128), 128),
    "cf112": (ConvFirst(8, 3), TensorDims(128, 112, 112, 16), None),
    "cf56": (ConvFirst(8, 6), TensorDims(128, 56, 56, 32), None),
    "cf28": (ConvFirst(8, 6), TensorDims(128, 28, 28, 48), None),
    "cf96": (ConvFirst(8, 6), TensorDims(8, 56, 56, 96), None),
    "cfs2_112": (ConvFirst(8, 6, 2), TensorDims(128, 112, 112, 16), 32),
    "cfs2_56": (ConvFirst(8, 6, 2), TensorDims(128, 56, 56, 32), 48),
    "nano_s2b0": (ConvFirst(8, 6, 2), TensorDims(128, 112, 112, 32), 48),
    "nano_s3b0": (ConvFirst(8, 6, 2), TensorDims(128, 56, 56, 48), 64),
    "small_s3b0": (ConvFirst(8, 6, 2), TensorDims(128, 56, 56, 64), 96),
    "stem": (Stem(16), TensorDims(128, 224, 224, 3), None),
    "head": (Head(1280, 1000), TensorDims(128, 7, 7, 128), None),
    "cnx": (ConvNeXtBlock(), TensorDims(8, 56, 56, 96), None),
    "mbc2": (MBConv(1, 4, 0.25), TensorDims(128, 28, 28, 80), None),
    # ConvNeXt-T units at b128
    "cnx_stem": (PatchifyStem(96), TensorDims(128, 224, 224, 3), None),
    "cnx96": (ConvNeXtBlock(), TensorDims(128, 56, 56, 96), None),
    "cnx_ds1": (Downsample(192), TensorDims(128, 56, 56, 96), None),
    "cnx192": (ConvNeXtBlock(), TensorDims(128, 28, 28, 192), None),
    "cnx384": (ConvNeXtBlock(), TensorDims(128, 14, 14, 384), None),
    "cnx768": (ConvNeXtBlock(), TensorDims(128, 7, 7, 768), None),
    "cnx_head": (LNHead(1000), TensorDims(128, 7, 7, 768), None),
    "ffn384": (FFN(4, "gelu"), TensorDims(128, 14, 14, 384), None),
}
ap = argparse.ArgumentParser(); ap.add_argument("names", nargs="+"); ap.add_argument("--iters", type=int, default=3); ap.add_argument("--timed", type=int, default=50)
a = ap.parse_args()
for nm in a.names:
    blk, dims, k = CASES[nm]
    m = FusedBlock(blk, dims, k)
    x = torch.randn(*m.in_shape, device="cuda").half()
    out = torch.empty(m.out_shape, dtype=torch.float16, device="cuda")
    for _ in range(a.iters):
        m.launch(x, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if a.timed < 1:
        continue
    e0.record()
    for _ in range(a.timed): m.launch(x, out)
    e1.record(); e1.synchronize()
    print(nm, "%.1f us" % (e0.elapsed_time(e1) / a.timed * 1e3), flush=True)
