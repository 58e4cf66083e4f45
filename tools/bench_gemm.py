"""Sweep of the tcgen05 GEMM (wl_gemm): time per call (CUDA events, 20 calls) and TFLOP/s."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_03617_b200 import _lib
_lib.lib().wl_init(0)
shapes = [(27264, 192, 768, "gelu", False), (27264, 192, 768, "identity", False), (27264, 768, 192, "identity", True),
          (25088, 384, 1536, "gelu", False), (25088, 1536, 384, "identity", True), (8192, 4096, 4096, "identity", False),
          (16384, 1024, 1024, "identity", False), (401408, 48, 96, "identity", False), (27264, 64, 256, "identity", False)]
for m, k, n, act, res in shapes:
    a = torch.randn(m, k, device="cuda").half(); b = torch.randn(n, k, device="cuda").half() / k ** 0.5
    bias = torch.randn(n, device="cuda"); r = torch.randn(m, n, device="cuda").half() if res else None
    out = _lib.gemm(a, b, bias, act, r)
    ref = (a.float() @ b.float().T + bias)
    if act == "gelu": ref = torch.nn.functional.gelu(ref)
    if res: ref = ref + r.float()
    err = ((out.float() - ref).abs().max() / ref.abs().max()).item()
    for _ in range(3): _lib.gemm(a, b, bias, act, r, out=out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): _lib.gemm(a, b, bias, act, r, out=out)
    e1.record(); e1.synchronize()
    t = e0.elapsed_time(e1) / 20 / 1e3
    print(f"M={m:6d} K={k:5d} N={n:5d} {act:8s} res={res:d}: {t*1e6:8.1f} us {2*m*n*k/t/1e12:7.1f} TF/s  err {err:.1e}", flush=True)
