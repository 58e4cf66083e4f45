"""One small launch per kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck). Usage: python tools/sanitize_cases.py [case ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_03617_b200.blocks import FusedBlock  # noqa: E402
from paper_2404_03617_b200.core import (  # noqa: E402
    FFN, ConvFirst, ConvNeXtBlock, ExecutionScheme, Head, MBConv, Stem, TensorDims)

CASES = {
    "cf_fused": (ConvFirst(8, 6), TensorDims(1, 20, 12, 32), None),
    "cf_convnext": (ConvNeXtBlock(7, 4, "gelu"), TensorDims(1, 16, 16, 96), None),
    "cf_s2": (ConvFirst(8, 6, 2), TensorDims(1, 56, 56, 32), 48),
    "mb_s1_14": (MBConv(8, 4, 0.25), TensorDims(2, 14, 14, 128), None),
    "mb_s1_7": (MBConv(8, 4, 0.25), TensorDims(2, 7, 7, 128), None),
    "mb_front_pair": (MBConv(8, 4, 0.25), TensorDims(2, 14, 14, 256), None),
    "mb_front_s2": (MBConv(8, 4, 0.25, 2), TensorDims(1, 28, 28, 48), 128),
    "mb_front_t1": (MBConv(1, 4, 0.25), TensorDims(1, 28, 28, 80), None),
    "stem": (Stem(16), TensorDims(1, 64, 48, 3), None),
    "head": (Head(1280, 1000), TensorDims(2, 7, 7, 128), None),
    # round 2
    "mb_s1_s2": (MBConv(8, 4, 0.25, 2), TensorDims(2, 14, 14, 128), 128),
    "cf_wide": (ConvFirst(8, 6), TensorDims(1, 14, 14, 192), None),
    "ffn": (FFN(4, "gelu"), TensorDims(1, 14, 14, 96), None),
    "lw_mbconv": (MBConv(8, 4, 0.25), TensorDims(2, 7, 7, 128), None),
    "lw_convfirst": (ConvFirst(8, 6), TensorDims(1, 14, 14, 32), None),
    # session 3: dwln7 + the fused FFN (C = 192 route, C = 96 direct stores with the residual
    # prefetch at 65536 pixels) and the two GEMMs (C = 384)
    "cnx_c192": (ConvNeXtBlock(7, 4, "gelu"), TensorDims(1, 14, 14, 192), None),
    "cnx_c96_big": (ConvNeXtBlock(7, 4, "gelu"), TensorDims(21, 56, 56, 96), None),
    "cnx_c384": (ConvNeXtBlock(7, 4, "gelu"), TensorDims(1, 14, 14, 384), None),
}
LAYER_WISE = {"lw_mbconv", "lw_convfirst"}
names = sys.argv[1:] or list(CASES) + ["mb_stage"]
for nm in names:
    if nm == "mb_stage":  # per-stage persistent launch: two 7x7 blocks in one launch
        from paper_2404_03617_b200 import zoo
        from paper_2404_03617_b200.scheduler import FusedNetwork

        net = FusedNetwork(zoo.build_stack(MBConv(8, 4, 0.25), 3, TensorDims(2, 7, 7, 128)), batch=2, seed=1)
        net.x.normal_()
        net.launch_all()
        torch.cuda.synchronize()
        print(nm, "ok", [k for _, _, k in net.steps], flush=True)
        continue
    blk, dims, k = CASES[nm]
    m = FusedBlock(blk, dims, k, scheme=ExecutionScheme.LAYER_WISE if nm in LAYER_WISE else ExecutionScheme.BLOCK_FUSION)
    x = torch.randn(*m.in_shape, device="cuda").half()
    out = torch.empty(m.out_shape, dtype=torch.float16, device="cuda")
    m.launch(x, out)
    torch.cuda.synchronize()
    print(nm, "ok", flush=True)
