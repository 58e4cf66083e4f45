import glob, json, sys, os, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_03617_b200 import _lib as L

def desc_cf(meta, act):
    d = L.BlockDesc()
    n, h, w, c = meta["dims"]; p = meta["params"]
    d.kind = L.KIND_CONVFIRST; d.n, d.h, d.w, d.c, d.k = n, h, w, c, c
    d.expansion = p["expansion"]; d.group_width = p["group_width"]; d.ksize = 3; d.stride = 1
    d.act = L.ACTS[p["activation"]]
    return d

fails = 0
for f in sorted(glob.glob("tests/golden/convfirst*.npz")):
    z = np.load(f); meta = json.loads(str(z["meta"]))
    if meta["dims"][3] % 16: print("skip", f); continue
    d = desc_cf(meta, None)
    names = ["w_conv", "b_conv", "u", "a", "v", "b"]
    ws = [z["in_" + k].astype(np.float32) for k in names]
    x = z["in_x"].astype(np.float32)
    try:
        out = L.execute_numeric_host(d, x, ws)
    except Exception as e:
        print("ERR", f, e); fails += 1; continue
    ref = z["out_layerwise"]
    err = np.abs(out - ref).max() / np.abs(ref).max()
    l2 = np.linalg.norm(out - ref) / np.linalg.norm(ref)
    ok = err < 1e-2 and l2 < 2e-3
    fails += not ok
    print(os.path.basename(f), "maxrel %.3g l2rel %.3g" % (err, l2), "OK" if ok else "FAIL")
print("FAILS", fails)

# ---------------- MBConv golden
def desc_mb(meta):
    d = L.BlockDesc()
    n, h, w, c = meta["dims"]; p = meta["params"]
    d.kind = L.KIND_MBCONV; d.n, d.h, d.w, d.c, d.k = n, h, w, c, c
    d.expansion = p["expansion"]; d.group_width = p["group_width"]; d.ksize = 3; d.stride = 1
    d.se_sq = int(p["se_ratio"] * c); d.act = L.ACTS[p["activation"]]
    return d
fails = 0
for f in sorted(glob.glob("tests/golden/mbconv*.npz")):
    z = np.load(f); meta = json.loads(str(z["meta"]))
    d = desc_mb(meta)
    names = ["w_exp", "b_exp", "w_conv", "b_conv", "w_sq", "b_sq", "w_ex", "b_ex", "w_prj", "b_prj"]
    ws = [z["in_" + k].astype(np.float32) for k in names]
    x = z["in_x"].astype(np.float32)
    try:
        out = L.execute_numeric_host(d, x, ws)
    except Exception as e:
        print("ERR", f, e); fails += 1; continue
    ref = z["out_layerwise"]
    err = np.abs(out - ref).max() / np.abs(ref).max()
    l2 = np.linalg.norm(out - ref) / np.linalg.norm(ref)
    ok = err < 1e-2 and l2 < 2e-3
    fails += not ok
    print(os.path.basename(f), "maxrel %.3g l2rel %.3g" % (err, l2), "OK" if ok else "FAIL")
print("MB FAILS", fails)
