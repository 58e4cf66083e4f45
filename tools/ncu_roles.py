"""Attribute ncu stall samples of a warp-specialised kernel to its roles:
python tools/ncu_roles.py report.ncu-rep kernel_file.cu 'role:first-last,...'
(role line ranges in kernel_file.cu; inlined header code is attributed to the
role of the nearest preceding kernel-file instruction in address order)."""

import csv
import io
import subprocess
import sys
from collections import defaultdict


def main(rep, kfile, spec):
    roles = []
    for part in spec.split(","):
        name, rng = part.split(":")
        a, b = rng.split("-")
        roles.append((name, int(a), int(b)))
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, cline, hdr = None, None, None
    ins = []  # (addr, file, line, samples, notissued, sass)
    for r in csv.reader(io.StringIO(txt)):
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 6:
            continue
        if r[0] != "":
            cline = int(r[0])
            continue
        try:
            ins.append((int(r[2], 16), cur, cline, int(r[4]), int(r[5]), r[3].strip()))
        except ValueError:
            pass
    ins.sort()
    role_of = lambda ln: next((n for n, a, b in roles if a <= ln <= b), "other")
    last = "other"
    agg = defaultdict(lambda: [0, 0])
    top = defaultdict(lambda: defaultdict(int))
    for addr, f, ln, s, ni, sass in ins:
        if f == kfile:
            last = role_of(ln)
        agg[last][0] += s
        agg[last][1] += ni
        top[last][f"{f}:{ln} {sass.split()[0] if sass else ''}"] += s
    tot = sum(v[0] for v in agg.values())
    for k, (s, ni) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{k:10s} {s:7d} samples ({100 * s / tot:5.1f}%), not issued {ni}")
        for key, v in sorted(top[k].items(), key=lambda kv: -kv[1])[:8]:
            print(f"      {v:6d}  {key}")


if __name__ == "__main__":
    main(*sys.argv[1:4])
