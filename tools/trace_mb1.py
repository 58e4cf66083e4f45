"""Phase timeline of CTA 0 of the stride-1 MBConv kernel (mb_s1.cu, clock64 stamps)."""
import sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_03617_b200 import _lib
from paper_2404_03617_b200.core import MBConv, TensorDims
from paper_2404_03617_b200.blocks import FusedBlock
for h in [int(v) for v in (sys.argv[1:] or ["14", "7"])]:
    dims = TensorDims(128, h, h, 128)
    m = FusedBlock(MBConv(8, 4, 0.25), dims)
    x = torch.randn(dims.n, dims.h, dims.w, dims.c, device="cuda").half()
    out = torch.empty(m.out_shape, dtype=torch.float16, device="cuda")
    buf = torch.zeros(4608, dtype=torch.int64, device="cuda")
    for _ in range(3): m.launch(x, out)
    _lib.lib().wl_debug_set_trace(buf.data_ptr())
    m.launch(x, out)
    torch.cuda.synchronize()
    _lib.lib().wl_debug_set_trace(None)
    t = buf.cpu().tolist()
    r = lambda v: (v - t[0]) if v else -1
    print(f"mb{h}: x@{r(t[70])} convA_end@{r(t[1])} SE_end@{r(t[2])} gate_end@{r(t[3])} z_full@{r(t[68])} stored@{r(t[69])}")
    for j in range(8):
        print(f"  chunk {j}: expand@{r(t[36 + j])} h1_full@{r(t[4 + j])} conv_start@{r(t[12 + j])} "
              f"top@{r(t[72 + j])} ldg_issued@{r(t[80 + j])} mma_epi_done@{r(t[28 + j])} conv_done@{r(t[20 + j])} squeeze_done@{r(t[44 + j])} proj@{r(t[52 + j])}")

