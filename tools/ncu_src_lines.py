"""Top CUDA source lines by warp-stall samples of an ncu report (cuda,sass source page):
python tools/ncu_src_lines.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys


def main(rep, n=40):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, hdr, out = None, None, {}
    for r in csv.reader(io.StringIO(txt)):
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 6 or r[0] == "":
            continue
        try:
            out[(cur, r[0])] = (int(r[4]), int(r[5]), r[1][:100])
        except ValueError:
            pass
    tot = sum(v[0] for v in out.values())
    print("total samples", tot)
    for k, v in sorted(out.items(), key=lambda kv: -kv[1][0])[:n]:
        print(f"{v[0]:6d} {100 * v[0] / max(tot, 1):5.1f}% {v[1]:6d} {k[0]}:{k[1]} {v[2]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
