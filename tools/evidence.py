"""Summaries for profiles/: launch shares of an ncu launch list and key metrics
of ncu --set full reports.
  python tools/evidence.py shares launches.csv "header line"
  python tools/evidence.py ncu name=report.ncu-rep ..."""
import csv
import io
import re
import subprocess
import sys
from collections import OrderedDict


def shares(path, header):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    ui = h.index("Metric Unit")
    agg = OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[ki]).strip()
        if not name.startswith(("void wl::", "wl::")):
            continue
        a = agg.setdefault(name[:52], [0, 0.0])
        a[0] += 1
        scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(r[ui], 1.0)
        a[1] += float(r[vi].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values())
    print(header)
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:52s} {n:3d} launches {t:9.1f} us {100 * t / tot:5.1f}%")


KEYS = [
    ("duration_us", "gpu__time_duration.sum"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
    ("regs", "launch__registers_per_thread"),
    ("smem_dyn_KB", "launch__shared_mem_per_block_dynamic"),
    ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("hmma_pipe_pct", "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active"),
    ("tensor_pipe_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("dram_read_MB", "dram__bytes_read.sum"),
    ("dram_write_MB", "dram__bytes_write.sum"),
    ("smem_bank_conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    ("warp_instr", "smsp__inst_executed.sum"),
]


def ncu(items):
    for it in items:
        name, rep = it.split("=", 1)
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(txt)))
        if len(rows) < 3:
            print(f"== {name}: no data")
            continue
        d = dict(zip(rows[0], rows[2]))
        print(f"== {name} ({d.get('Kernel Name', '')[:70]})")
        for k, m in KEYS:
            print(f"  {k:20s} {d.get(m, 'n/a')}")
        st = sorted(((float(d[k].replace(",", "")), k) for k in rows[0]
                     if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued") and d.get(k) not in ("", "n/a")),
                    reverse=True)
        print("  top stalls: " + ", ".join(f"{k.split('stalled_')[1]}={v:.0f}" for v, k in st[:6]))


if __name__ == "__main__":
    if sys.argv[1] == "shares":
        shares(sys.argv[2], sys.argv[3])
    else:
        ncu(sys.argv[2:])
