"""Per-source-line stall breakdown of an ncu report (cuda source page):
python tools/ncu_line_stalls.py report.ncu-rep file.cu line [line ...]  (no lines: the top 15 lines)"""
import csv
import io
import subprocess
import sys

rep, fname = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None
want = set(sys.argv[3:])
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True,
                     text=True).stdout
cur, hdr, rows = None, None, []
for r in csv.reader(io.StringIO(txt)):
    if len(r) >= 2 and r[0] == "File Name":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit() and hdr[0] == "Line No":
        rows.append((cur, dict(zip(hdr, r))))
stalls = [h for h in (hdr or []) if h.startswith("stall_") and "Not Issued" not in h]
rows = [(f, d) for f, d in rows if (fname is None or f == fname) and (not want or d["Line No"] in want)]
rows.sort(key=lambda fd: -int(fd[1]["Warp Stall Sampling (All Samples)"] or 0))
for f, d in rows[:15 if not want else len(rows)]:
    tot = int(d["Warp Stall Sampling (All Samples)"] or 0)
    top = sorted(((int(d[s] or 0), s[6:]) for s in stalls), reverse=True)[:4]
    print(f"{f}:{d['Line No']:>5} {tot:6d}  " + "  ".join(f"{n}={v}" for v, n in top if v) + f"   | {d['Source'].strip()[:70]}")
