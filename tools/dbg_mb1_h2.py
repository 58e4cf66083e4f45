"""Compare the stride-1 MBConv kernel's h2 (conv output, read back from the
workspace) with the oracle's, per row / column / channel."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import blocks as B
from paper_2404_03617_b200.core import MBConv, TensorDims
from paper_2404_03617_b200.blocks import FusedBlock
from paper_2404_03617_b200.machine import build_schedule, random_inputs
h = int(sys.argv[1]) if len(sys.argv) > 1 else 7
dims = TensorDims(1, h, h, 128)
s = build_schedule(MBConv(8, 4, 0.25), dims)
ins = {k: v.astype(np.float16).astype(np.float32) for k, v in random_inputs(s, np.random.default_rng(0), 0.3).items()}
w = {k: v for k, v in ins.items() if k != "x"}
m = FusedBlock(s.block, dims, weights=w)
x = torch.from_numpy(ins["x"]).half().cuda()
out = torch.empty(m.out_shape, dtype=torch.float16, device="cuda")
m.workspace.zero_()
m.launch(x, out)
torch.cuda.synchronize()
NT = (16 * h + 127) // 128
ws = m.workspace.cpu().numpy()[4096:]
hid = 512
nch = hid // 64
raw = ws[: nch * NT * 16384].view(np.float16).reshape(nch, NT, 8, 128, 8).astype(np.float32)
# -> flat rows m (NT*128), channels (nch*64)
h2 = raw.transpose(1, 3, 0, 2, 4).reshape(NT * 128, hid)
h1r = B._f32(B.phi("silu", B._f32(B._mm(ins["x"], ins["w_exp"], ins["b_exp"]))))
h2r = B._f32(B.phi("silu", B._f32(B.grouped_conv2d(h1r, ins["w_conv"], ins["b_conv"]))))[0]
got = np.zeros((h, h, hid), np.float32)
for y in range(h):
    for xx in range(h):
        got[y, xx] = h2[y * 16 + xx + 1]
err = np.abs(got - h2r)
sc = np.abs(h2r).max()
np.set_printoptions(precision=3, linewidth=220)
print("h2 max rel", err.max() / sc, "ref max", sc, "got max", np.abs(got).max())
print("by row", err.max(axis=(1, 2)) / sc)
print("by col", err.max(axis=(0, 2)) / sc)
print("by ch%8", (err.max(axis=(0, 1)) / sc).reshape(-1, 8).max(0))
print("by group (first 16)", (err.max(axis=(0, 1)) / sc).reshape(-1, 8).max(1)[:16])
print("pad rows nonzero:", [i for i in range(16) if np.abs(h2[i::16][:h]).max() > 0 and (i == 0 or i > h)])
# is h2 off by a shift? test shifts of the oracle
for dy in (-1, 0, 1):
    for dx in (-1, 0, 1):
        sh = np.zeros_like(got)
        for y in range(h):
            for xx in range(h):
                yy, xs = y + dy, xx + dx
                if 0 <= yy < h and 0 <= xs < h:
                    sh[y, xx] = h2r[yy, xs]
        print("shift", dy, dx, "err", np.abs(got - sh)[1:-1, 1:-1].max() / sc)
