"""Localise a parity error of the stride-1 MBConv kernel: error by row, column, channel.
usage: python tools/dbg_mb1.py H [tensor,tensor...]   (listed weight tensors are zeroed)"""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2404_03617_b200.core import MBConv, TensorDims
from paper_2404_03617_b200.machine import build_schedule, execute_numeric, random_inputs
h = int(sys.argv[1]) if len(sys.argv) > 1 else 7
zero = sys.argv[2].split(",") if len(sys.argv) > 2 else []
dims = TensorDims(1, h, h, 128)
s = build_schedule(MBConv(8, 4, 0.25), dims)
ins = {k: v.astype(np.float16).astype(np.float32) for k, v in random_inputs(s, np.random.default_rng(0), 0.3).items()}
for z in zero:
    ins[z] = np.zeros_like(ins[z])
got = execute_numeric(s, ins)
ref = oracle.mbconv_block(*[ins[k] for k in ("x", "w_exp", "b_exp", "w_conv", "b_conv", "w_sq", "b_sq", "w_ex", "b_ex",
                                             "w_prj", "b_prj")])
err = np.abs(got - ref)[0]
sc = np.abs(ref).max()
np.set_printoptions(precision=3, linewidth=200)
print("zeroed", zero, "max rel", err.max() / sc)
print("by row", err.max(axis=(1, 2)) / sc)
print("by col", err.max(axis=(0, 2)) / sc)
print("by ch%64", (err.max(axis=(0, 1)) / sc).reshape(-1, 64).max(0))
