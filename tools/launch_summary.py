"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import re
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        v = v / 1000.0 if u in ("nsecond", "ns") else v * 1000.0 if u in ("msecond", "ms") else v
        agg[re.sub(r"\(.*", "", r[ki])[:60]][0] += 1
        agg[re.sub(r"\(.*", "", r[ki])[:60]][1] += v
    tot = sum(a[1] for a in agg.values())
    print(f"total {tot:.1f} us over {sum(a[0] for a in agg.values())} launches")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:55s} n={n:5d} tot={t:9.1f}us avg={t / n:7.2f}us share={t / tot:.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
