"""One wl_gemm call for ncu: python tools/prof_gemm.py M K N act [res]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_03617_b200 import _lib
_lib.lib().wl_init(0)
m, k, n, act = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
res = len(sys.argv) > 5
a = torch.randn(m, k, device="cuda").half(); b = torch.randn(n, k, device="cuda").half() / k ** 0.5
bias = torch.randn(n, device="cuda"); r = torch.randn(m, n, device="cuda").half() if res else None
for _ in range(2): out = _lib.gemm(a, b, bias, act, r)
torch.cuda.synchronize()
