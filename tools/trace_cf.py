"""Tile timeline of CTA 0 of the stride-1 ConvFirst kernel (clock64 stamps)."""
import sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_03617_b200 import _lib
from paper_2404_03617_b200.core import ConvFirst, TensorDims
from paper_2404_03617_b200.blocks import FusedBlock
cases = {"cf112": (ConvFirst(8, 3), TensorDims(128, 112, 112, 16)),
         "cf56": (ConvFirst(8, 6), TensorDims(128, 56, 56, 32)),
         "cf28": (ConvFirst(8, 6), TensorDims(128, 28, 28, 48)),
         "cf96": (ConvFirst(8, 6), TensorDims(8, 56, 56, 96))}
names = ["halo", "cv_go", "cv_iss", "cepi", "cepi_e", "ffn", "H", "H_e", "prj", "fin", "fin_e"]
for nm in sys.argv[1:]:
    blk, dims = cases[nm]
    m = FusedBlock(blk, dims)
    x = torch.randn(dims.n, dims.h, dims.w, dims.c, device="cuda").half()
    out = torch.empty(m.out_shape, dtype=torch.float16, device="cuda")
    buf = torch.zeros(256, dtype=torch.int64, device="cuda")
    for _ in range(3): m.launch(x, out)
    _lib.lib().wl_debug_set_trace(buf.data_ptr())
    m.launch(x, out)
    torch.cuda.synchronize()
    _lib.lib().wl_debug_set_trace(None)
    t = buf.cpu().tolist()
    t0 = t[0]
    rel = lambda v: (v - t0) if v else -1
    print(nm, "halo_bufs*100+nchunks", t[2], "r", t[3])
    for i in range(16):
        row = t[8 + 12 * i: 8 + 12 * i + 11]
        print(f" tile {i:2d}: " + " ".join(f"{n}={rel(v)}" for n, v in zip(names, row)))
