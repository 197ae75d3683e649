"""DRAM bytes per launch by bench kernel class, from an ncu --csv launch list
(metrics gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum;
ncu's default cache control, i.e. cold caches per launch). Solve-phase
launches only (from the first k_spmv_dots). Updates profiles/ncu_summary.json:
  python tools/ncu_class_traffic.py launches.csv cfg0"""
import collections
import csv
import json
import os
import re
import sys

CLASSES = [  # first match wins; mirrors the ProfScope classes in csrc/fsigpu.cu
    ("block_solve", r"EpiAxpy|EpiSetScaled|block_solve|inv_gemv|fs_combine"),
    ("transfer", r"prolong_resid|EpiRestrict|EpiProlong"),
    ("coarse", r"gemv_kernel"),
    ("arnoldi", r"k_update|k_norm|k_cycle|k_solve_y|givens"),
    ("spmv", r"k_spmv_dots|csr_kernel|csr_pair_kernel"),
]


def main(path, config):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ci = {n: h.index(n) for n in ["ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"]}
    launches = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= ci["Metric Value"]:
            continue
        d = launches.setdefault(r[ci["ID"]], {"name": r[ci["Kernel Name"]], "bytes": 0.0})
        if r[ci["Metric Name"]].startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[ci["Metric Unit"]], 1)
            d["bytes"] += float(r[ci["Metric Value"]].replace(",", "")) * scale
    seq = list(launches.values())
    first = next((i for i, d in enumerate(seq) if "k_spmv_dots" in d["name"] or "k_cycle_start" in d["name"]), 0)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in seq[first:]:
        for cls, pat in CLASSES:
            if re.search(pat, d["name"]):
                agg[cls][0] += 1
                agg[cls][1] += d["bytes"]
                break
    out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                            "ncu_summary.json")
    js = json.load(open(out_path)) if os.path.exists(out_path) else {}
    js.setdefault("dram_bytes_per_launch", {})
    for cls, (n, b) in agg.items():
        js["dram_bytes_per_launch"][f"{cls}@{config}"] = b / n
    js["source"] = ("tools/ncu_class_traffic.py over ncu launch lists (gpu__time_duration, dram bytes; cold caches "
                    "per launch): DRAM bytes per launch averaged over the solve-phase launches of each class")
    json.dump(js, open(out_path, "w"), indent=1)
    print(json.dumps(js, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
