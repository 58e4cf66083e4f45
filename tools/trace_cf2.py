"""Phase timeline of CTA 0 of the stride-2 ConvFirst kernel (clock64 stamps)."""
import sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_03617_b200 import _lib
from paper_2404_03617_b200.core import ConvFirst, TensorDims
from paper_2404_03617_b200.blocks import FusedBlock
cases = {"cfs2_112": (ConvFirst(8, 6, 2), TensorDims(128, 112, 112, 16), 32),
         "cfs2_56": (ConvFirst(8, 6, 2), TensorDims(128, 56, 56, 32), 48)}
for nm in sys.argv[1:]:
    blk, dims, k = cases[nm]
    m = FusedBlock(blk, dims, k)
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
    print(nm, "R*1000+r", t[2], "nct/neh/npt", t[3], "nb*10+xbufs", t[4], "end", rel(t[1]))
    names = ["xload", "cv_wait", "cv_go", "cv_iss", "xh_ok", "ffn_iss", "G1cv", "G1drn", "G1xh",
             "E0", "y0", "q0", "E1", "y1", "q1", "E2", "y2", "q2", "E3", "y3", "q3", "Z", "Zd"]
    for i in range(8):
        row = t[8 + 24 * i: 8 + 24 * i + 23]
        print(f" band {i}: " + " ".join(f"{n}={rel(v)}" for n, v in zip(names, row)))
