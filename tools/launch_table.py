"""Per-kernel table from an ncu --csv launch list with gpu__time_duration.sum and
dram__bytes_{read,write}.sum. Only launches after the first Arnoldi kernel
(k_spmv_dots) count, i.e. the solve, not the setup. Kernels are keyed by name
+ grid size (grid size separates the levels of the hierarchy).
Usage: python tools/launch_table.py launches.csv"""
import collections
import csv
import re
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    col = {n: h.index(n) for n in ["ID", "Kernel Name", "Grid Size", "Metric Name", "Metric Unit", "Metric Value"]}
    launches = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= col["Metric Value"]:
            continue
        lid = r[col["ID"]]
        d = launches.setdefault(lid, {"name": r[col["Kernel Name"]], "grid": r[col["Grid Size"]]})
        v = float(r[col["Metric Value"]].replace(",", ""))
        u = r[col["Metric Unit"]]
        m = r[col["Metric Name"]]
        if m.startswith("gpu__time_duration"):
            d["us"] = v / 1000.0 if u in ("nsecond", "ns") else v * 1000.0 if u in ("msecond", "ms") else v
        elif m.startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            d["bytes"] = d.get("bytes", 0.0) + v * scale
    seq = list(launches.values())
    first = next((i for i, d in enumerate(seq) if "k_spmv_dots" in d["name"] or "k_cycle_start" in d["name"]), 0)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in seq[first:]:
        base = re.sub(r"\(.*", "", d["name"])
        epi = re.findall(r"Epi\w+|Gather\w+", d["name"])
        key = f"{base[:28]} {'/'.join(epi)[:34]} g={d['grid']}"
        a = agg[key]
        a[0] += 1
        a[1] += d.get("us", 0.0)
        a[2] += d.get("bytes", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"solve-phase launches: {sum(a[0] for a in agg.values())}, total {tot / 1000:.2f} ms (serialised, cold)")
    print(f"{'kernel':80s} {'n':>5s} {'avg us':>8s} {'share':>6s} {'DRAM MB/launch':>14s} {'GB/s':>7s}")
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:80s} {n:5d} {t / n:8.1f} {t / tot:6.3f} {b / n / 1e6:14.1f} {b / t / 1e3 if t else 0:7.0f}")


if __name__ == "__main__":
    main(sys.argv[1])
