"""Top CUDA source lines by warp-stall samples from an ncu report
(aggregates the `--page source --print-source=cuda,sass` export per line)."""
import csv, subprocess, sys, io, collections
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = None; hdr = None
agg = collections.defaultdict(lambda: collections.Counter()); src = {}
key = "Warp Stall Sampling (All Samples)"
for r in rows:
    if not r: continue
    if r[0] in ("File Path", "File Name"): fname = r[1].split("/")[-1]; hdr = None; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr and len(r) == len(hdr):
        ln = (fname, r[0]); src[ln] = r[1]
        for i, c in enumerate(hdr):
            if i >= 4 and (c == key or (c.startswith("stall_") and "Not Issued" not in c)):
                try: agg[ln][c] += float(r[i] or 0)
                except ValueError: pass
tot = sum(v[key] for v in agg.values()) or 1
for ln, v in sorted(agg.items(), key=lambda kv: -kv[1][key])[:n]:
    st = sorted(((c[6:], x) for c, x in v.items() if c.startswith("stall_")), key=lambda x: -x[1])[:2]
    print(f"{100*v[key]/tot:5.1f}% {ln[0]}:{ln[1]:>5} {src[ln].strip()[:70]:70s} {[(a, int(b)) for a, b in st]}")
