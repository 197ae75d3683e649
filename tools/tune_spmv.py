"""Sweep SpMV launch shapes (lanes per row x batch depth) on one hierarchy.

usage: tune_spmv.py [data.fsix] [level ...]   (default: every level >= 1)
FSI_WHICH=A,R limits the sweep to those matrices. FSI_WARM=1 times back-to-back launches (L2-resident, the in-solve regime of
small hierarchies) instead of launches after an L2 flush.
"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_13201_b200 import fsigpu
from paper_1909_13201_b200.problem import load_case
fsigpu.init(0)
path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "data", "cfg0.fsix")
P = load_case(path)
G = fsigpu.GmgPreconditioner(P.levels)
levels = [int(a) for a in sys.argv[2:]] or list(range(1, len(P.levels)))
cold = os.environ.get("FSI_WARM", "0") != "1"
for lev in levels:
    L = P.levels[lev]
    kinds = [("A", "residual"), ("FS", "fs_smoother"), ("AP", "prolong_resid"), ("R", "restrict")]
    only = os.environ.get("FSI_WHICH")
    for which, kname in kinds:
        if only and which not in only.split(","):
            continue
        best, default = None, None
        default = G.time_kernel(kname, lev, reps=10, cold=cold)[0]
        for lpr in [1, 2, 4, 8, 16, 32]:
            for u in [4, 8, 22, 24]:
                if lpr == 1 and u < 22:
                    continue
                G.set_launch(lev, which, lpr, u)
                ms, by = G.time_kernel(kname, lev, reps=10, cold=cold)
                if best is None or ms < best[0]:
                    best = (ms, lpr, u, by)
        print(f"L{lev} n={L.n:8d} nnz/row={(L.R.nnz / L.R.rows if which == "R" else L.A.nnz / L.n):5.1f} {which:3s} default {default*1000:8.2f} us  best lpr={best[1]:2d} u={best[2]} "
              f"{best[0]*1000:8.2f} us {best[3]/best[0]/1e6:7.0f} GB/s", flush=True)
        G.set_launch(lev, which, best[1], best[2])
