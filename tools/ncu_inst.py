"""Executed warp instructions per source line from an ncu report (top N lines).
Usage: python tools/ncu_inst.py report.ncu-rep [N] [divide_by]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
div = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
res, cur, hdr = [], None, None
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) > 8 and r[0]:
        try:
            res.append((int(r[hdr.index("Instructions Executed")]), cur, r[0], r[1][:90]))
        except ValueError:
            pass
tot = sum(x[0] for x in res) or 1
print(f"total warp instructions {tot} ({tot / div:.0f} per unit)")
for x in sorted(res, reverse=True)[:n]:
    print(f"{100 * x[0] / tot:5.1f}% {x[0] / div:9.0f} {x[1]}:{x[2]}  {x[3]}")
