"""Per-source-line warp-stall samples from an ncu report (top N lines).
Usage: python tools/ncu_lines.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
res, cur, hdr = [], None, None
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) > 5 and r[0]:
        try:
            res.append((int(r[4]), int(r[5]), cur, r[0], r[1][:90]))
        except ValueError:
            pass
tot = sum(x[0] for x in res) or 1
print(f"total samples {tot}")
for x in sorted(res, reverse=True)[:n]:
    print(f"{100 * x[0] / tot:5.1f}% {x[0]:7d} (not-issued {x[1]:7d}) {x[2]}:{x[3]}  {x[4]}")
