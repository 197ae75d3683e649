"""Top stall locations (SASS) of an ncu report: python tools/ncu_hot.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys


def main(rep, n=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    si, wi = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    def num(x):
        try:
            float(x)
            return True
        except ValueError:
            return False
    body = [r for r in rows[2:] if len(r) > wi and num(r[wi] or "0")]
    tot = sum(float(r[wi] or 0) for r in body) or 1.0
    for idx, r in enumerate(body):
        r.append(idx)
    for r in sorted(body, key=lambda r: -float(r[wi] or 0))[:n]:
        print(f"{float(r[wi]) / tot:6.3f}  #{r[-1]:5d}  {r[si].strip()[:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
