import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_03617_b200 import _lib as L
import oracle

rng = np.random.default_rng(0)
def r(*s, scale=0.5):
    return (scale * rng.standard_normal(s)).astype(np.float16).astype(np.float32)
def cmp(name, out, ref):
    err = np.abs(out - ref).max() / np.abs(ref).max()
    l2 = np.linalg.norm(out - ref) / np.linalg.norm(ref)
    ok = err < 1e-2 and l2 < 2e-3
    print(f"{name}: maxrel {err:.3g} l2rel {l2:.3g} {'OK' if ok else 'FAIL'}", flush=True)
    return ok

fails = 0
# stem
for (n, H, W, Cs) in [(2, 32, 32, 16), (1, 224, 224, 16), (1, 224, 224, 24)]:
    d = L.BlockDesc(); d.kind = L.KIND_STEM; d.n, d.h, d.w, d.c, d.k = n, H, W, 3, Cs; d.act = 1; d.stride = 2
    x = r(n, H, W, 3, scale=1.0); w = r(Cs, 3, 3, 3); b = r(Cs)
    out = L.execute_numeric_host(d, x, [w, b])
    fails += not cmp(f"stem {n}x{H}x{W}->{Cs}", out, oracle.stem_block(x, w, b))
# cf2
for (n, H, W, C, K, a) in [(2, 16, 16, 16, 32, 6), (1, 112, 112, 16, 32, 6), (1, 56, 56, 32, 48, 6), (1, 28, 28, 48, 64, 6)]:
    d = L.BlockDesc(); d.kind = L.KIND_CONVFIRST; d.n, d.h, d.w, d.c, d.k = n, H, W, C, K
    d.expansion = a; d.group_width = 8; d.ksize = 3; d.stride = 2; d.act = 1
    hid = a * C
    x = r(n, H, W, C, scale=1.0); ws = [r(C, 3, 3, 8), r(C), r(C, hid, scale=0.5 / np.sqrt(C / 8)), r(hid), r(hid, K, scale=0.5 / np.sqrt(hid / 8)), r(K)]
    out = L.execute_numeric_host(d, x, ws)
    fails += not cmp(f"cf_s2 {n}x{H}x{W}x{C}->{K} a{a}", out, oracle.convfirst_s2_block(x, *ws))
# mbconv s2
for (n, H, W, C, K, a) in [(2, 28, 28, 48, 128, 4), (2, 14, 14, 128, 128, 4), (2, 16, 16, 32, 48, 4)]:
    d = L.BlockDesc(); d.kind = L.KIND_MBCONV; d.n, d.h, d.w, d.c, d.k = n, H, W, C, K
    d.expansion = a; d.group_width = 8; d.ksize = 3; d.stride = 2; d.act = 2; d.se_sq = int(0.25 * C)
    hid = a * C; sq = d.se_sq
    x = r(n, H, W, C, scale=1.0)
    ws = [r(C, hid, scale=0.5 / np.sqrt(C / 8)), r(hid), r(hid, 3, 3, 8), r(hid), r(hid, sq), r(sq), r(sq, hid), r(hid), r(hid, K, scale=0.5 / np.sqrt(hid / 8)), r(K)]
    out = L.execute_numeric_host(d, x, ws)
    fails += not cmp(f"mbconv_s2 {n}x{H}x{W}x{C}->{K}", out, oracle.mbconv_block(x, *ws, activation="silu", stride=2))
# mbconv s1 28x28x80 T=1 (config C2 shape at n=2)
for (n, H, W, C, T) in [(2, 28, 28, 80, 1), (2, 14, 14, 128, 8)]:
    d = L.BlockDesc(); d.kind = L.KIND_MBCONV; d.n, d.h, d.w, d.c, d.k = n, H, W, C, C
    d.expansion = 4; d.group_width = T; d.ksize = 3; d.stride = 1; d.act = 2; d.se_sq = int(0.25 * C)
    hid = 4 * C; sq = d.se_sq
    x = r(n, H, W, C, scale=1.0)
    ws = [r(C, hid, scale=0.5 / np.sqrt(C / 8)), r(hid), r(hid, 3, 3, T), r(hid), r(hid, sq), r(sq), r(sq, hid), r(hid), r(hid, C, scale=0.5 / np.sqrt(hid / 8)), r(C)]
    out = L.execute_numeric_host(d, x, ws)
    fails += not cmp(f"mbconv_s1 {n}x{H}x{W}x{C} T{T}", out, oracle.mbconv_block(x, *ws, activation="silu"))
# convnext-style (C1 shape at n=1)
for (n, H, W, C) in [(1, 56, 56, 96), (2, 14, 14, 32)]:
    d = L.BlockDesc(); d.kind = L.KIND_CONVFIRST; d.n, d.h, d.w, d.c, d.k = n, H, W, C, C
    d.expansion = 4; d.group_width = 1; d.ksize = 7; d.stride = 1; d.act = 4; d.norm = 1; d.ln_eps = 1e-6
    hid = 4 * C
    x = r(n, H, W, C, scale=1.0)
    ws = [r(C, 7, 7, 1, scale=0.1), r(C), (1 + r(C, scale=0.1)), r(C, scale=0.1), r(C, hid, scale=1 / np.sqrt(C)), r(hid), r(hid, C, scale=1 / np.sqrt(hid)), r(C)]
    out = L.execute_numeric_host(d, x, ws)
    ref = oracle.convnext_block(x, ws[0], ws[1], ws[4], ws[5], ws[6], ws[7], activation="gelu", ln_gamma=ws[2], ln_beta=ws[3])
    fails += not cmp(f"convnext {n}x{H}x{W}x{C}", out, ref)
# head
for (n, H, W, C) in [(4, 7, 7, 128), (130, 7, 7, 128)]:
    d = L.BlockDesc(); d.kind = L.KIND_HEAD; d.n, d.h, d.w, d.c, d.k = n, H, W, C, 1000
    d.embed = 1280; d.classes = 1000; d.act = 1
    x = r(n, H, W, C, scale=1.0)
    ws = [r(C, 1280, scale=1 / np.sqrt(C)), r(1280), r(1280, 1000, scale=1 / np.sqrt(1280)), r(1000)]
    out = L.execute_numeric_host(d, x, ws).reshape(n, 1000)
    fails += not cmp(f"head {n}x{H}x{W}x{C}", out, oracle.head_block(x, *ws))
print("FAILS", fails)
