"""Phase timeline of CTA 0 of the fused FFN kernel (ffn.cu, clock64 stamps):
per hidden chunk g: E issued, E seen by the epilogue, H handed back, P issued."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_03617_b200 import _lib
from paper_2404_03617_b200.blocks import FusedBlock
from paper_2404_03617_b200.core import FFN, TensorDims
for c, hw in [(int(v.split('x')[0]), int(v.split('x')[1])) for v in (sys.argv[1:] or ["96x56", "192x28", "384x14"])]:
    dims = TensorDims(128, hw, hw, c)
    m = FusedBlock(FFN(4, "gelu"), dims)
    x = torch.randn(*m.in_shape, device="cuda").half()
    out = torch.empty(m.out_shape, dtype=torch.float16, device="cuda")
    buf = torch.zeros(4096, dtype=torch.int64, device="cuda")
    for _ in range(3): m.launch(x, out)
    _lib.lib().wl_debug_set_trace(buf.data_ptr())
    m.launch(x, out)
    torch.cuda.synchronize()
    _lib.lib().wl_debug_set_trace(None)
    t = buf.cpu().tolist()
    t0 = t[15]
    r = lambda v: (v - t0) if v else -1
    nch = 4 * c // (128 if c <= 256 else 64)
    print(f"C={c} {hw}x{hw}: nch={nch}")
    for tile in range(3):
        print(f"  tile {tile}: z_full@{r(t[3000+2*tile])} z_drained@{r(t[3000+2*tile+1])}")
    for g in range(min(3 * nch, (3000 - 16) // 4)):
        e, p, es, hd = (r(t[16 + g * 4 + k]) for k in range(4))
        ei, pi = r(t[2000 + 2 * g]), r(t[2000 + 2 * g + 1])
        print(f"  g{g:3d}: E@{e:7d} Eissued@{ei:7d} Eseen@{es:7d} H@{hd:7d} P@{p:7d} Pissued@{pi:7d}")

