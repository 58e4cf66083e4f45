"""Phase timeline of CTA 0 of the MBConv front kernel (clock64 stamps)."""
import sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_03617_b200 import _lib
from paper_2404_03617_b200.core import MBConv, TensorDims
from paper_2404_03617_b200.blocks import FusedBlock
cases = {"mb14": (MBConv(8, 4, 0.25), TensorDims(128, 14, 14, 128), None),
         "mb7": (MBConv(8, 4, 0.25), TensorDims(128, 7, 7, 128), None),
         "mbs2": (MBConv(8, 4, 0.25, 2), TensorDims(128, 28, 28, 48), 128),
         "c2": (MBConv(1, 4, 0.25), TensorDims(128, 28, 28, 80), None)}
for nm in sys.argv[1:]:
    blk, dims, k = cases[nm]
    m = FusedBlock(blk, dims, k)
    x = torch.randn(dims.n, dims.h, dims.w, dims.c, device="cuda").half()
    out = torch.empty(m.out_shape, dtype=torch.float16, device="cuda")
    buf = torch.zeros(512 + 2048 + 2048, dtype=torch.int64, device="cuda")
    for _ in range(3): m.launch(x, out)
    _lib.lib().wl_debug_set_trace(buf.data_ptr())
    m.launch(x, out)
    torch.cuda.synchronize()
    _lib.lib().wl_debug_set_trace(None)
    t = buf.cpu().tolist()
    spans = [(t[512 + 2 * b], t[512 + 2 * b + 1]) for b in range(1024) if t[512 + 2 * b]]
    if spans:
        s0 = min(a for a, _ in spans)
        starts = sorted((a - s0) / 1e3 for a, _ in spans)
        ends = sorted((b - s0) / 1e3 for _, b in spans)
        durs = sorted((b - a) / 1e3 for a, b in spans)
        waits = [(t[2561 + 2 * b] - t[2560 + 2 * b]) / 1e3 for b in range(1024) if t[2560 + 2 * b]]
        if waits:
            w = sorted(waits)
            print(nm, f"pair squeeze barrier wait min/med/max {w[0]:.2f}/{w[len(w)//2]:.2f}/{w[-1]:.2f} us over {len(w)} CTAs")
        print(nm, f"CTAs {len(spans)}: start spread {starts[0]:.1f}..{starts[-1]:.1f} us, end {ends[0]:.1f}..{ends[-1]:.1f} us, "
              f"span min/med/max {durs[0]:.1f}/{durs[len(durs)//2]:.1f}/{durs[-1]:.1f} us")
    t0 = t[0]
    rel = lambda v: (v - t0) if v else -1
    print(nm, "plan sa/ring/h1b/eb", t[14], "cb/xt/HC/npt", t[15])
    print(nm, "producer start", rel(t[1]), "x loaded", rel(t[2]), "pool done", rel(t[8]), "SE start", rel(t[9]), "SE end", rel(t[10]),
          "proj start", rel(t[11]), "z stored", rel(t[12]), "end", rel(t[13]))
    for j in range(12):
        row = t[16 + 8 * j: 16 + 8 * j + 7]
        if not any(row): break
        print(f"  chunk {j}: wload@{rel(t[16 + 8 * j + 7])} xwait@{rel(t[232 + j])} expand@{rel(row[0])} conv@{rel(row[1])}..{rel(row[2])} Eepi {rel(row[3])}..{rel(row[4])} Cepi {rel(row[5])}..{rel(row[6])} pool@{rel(t[160 + j])} drain_end@{rel(t[300 + j])} blur_end@{rel(t[320 + j])}")
    print("  proj: a_full", [rel(v) for v in t[112:120]])
    print("  proj: a_ready", [rel(v) for v in t[96:104]])
    print("  proj: v_full", [rel(v) for v in t[104:112]])
    print("  SE: pool loaded", rel(t[124]), "squeezed", rel(t[125]), "| epi: z_full", rel(t[120]), "tiles", rel(t[121]), rel(t[122]), rel(t[123]))
    print("  proj: load issue", [rel(v) for v in t[88:96]])
    print("  gating chunk 3 per warp (pa_full ok, pt_empty ok, loop done, st done):", [[rel(t[200 + 4 * w + i]) for i in (3, 0, 1, 2)] for w in range(8)])
