"""Sweep SpMV launch shapes (lanes per row x batch depth) on one hierarchy."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_13201_b200 import fsigpu
from paper_1909_13201_b200.problem import load_case
fsigpu.init(0)
path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "data", "cfg0.fsix")
P = load_case(path)
G = fsigpu.GmgPreconditioner(P.levels)
top = len(P.levels) - 1
for which, kname in [("A", "residual"), ("FS", "fs_smoother"), ("AP", "prolong_resid")]:
    best = None
    for lpr in [4, 8, 16, 32]:
        for u in [4, 8]:
            G.set_launch(top, which, lpr, u)
            ms, by = G.time_kernel(kname, top, reps=10, cold=True)
            gb = by / ms / 1e6
            print(f"{which:3s} lpr={lpr:2d} u={u} cold {ms*1000:8.2f} us {gb:8.1f} GB/s", flush=True)
            if best is None or ms < best[0]:
                best = (ms, lpr, u)
    print(f"{which} best lpr={best[1]} u={best[2]} {best[0]*1000:.2f} us", flush=True)
