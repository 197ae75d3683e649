"""Staged (shared-memory CSR-stream) SpMV vs the vector kernel, per level.

usage: tune_stage.py [data.fsix] [level ...]   (default: every level >= 1)
Checks that staging leaves the V-cycle output unchanged to 1e-13 and sweeps
the per-CTA entry capacity for the residual (A), FS smoother and restriction.
"""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_13201_b200 import fsigpu
from paper_1909_13201_b200.problem import load_case
fsigpu.init(0)
path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "data", "cfg0.fsix")
P = load_case(path)
G = fsigpu.GmgPreconditioner(P.levels)
levels = [int(a) for a in sys.argv[2:]] or list(range(1, len(P.levels)))
z0 = G.apply(P.b)
for lev in range(1, len(P.levels)):
    for w in ("A", "FS", "R"):
        G.set_staging(lev, w, 2048)
z1 = G.apply(P.b)
print(f"staged vs vector V-cycle: rel diff {np.linalg.norm(z1 - z0) / np.linalg.norm(z0):.3e}", flush=True)
for lev in levels:
    L = P.levels[lev]
    for which, kname in [("A", "residual"), ("FS", "fs_smoother"), ("R", "restrict")]:
        res = []
        for cap in [0, 512, 1024, 2048, 4096, 8192]:
            G.set_staging(lev, which, cap)
            ms, by = G.time_kernel(kname, lev, reps=10, cold=True)
            msw, _ = G.time_kernel(kname, lev, reps=10, cold=False)
            res.append((cap, ms, msw, by))
        line = " ".join(f"{c}:{m*1000:.1f}/{mw*1000:.1f}" for c, m, mw, _ in res)
        best = min(res, key=lambda r: r[1])
        print(f"L{lev} n={L.n:8d} {which:2s} cold/warm us  {line}   best cap={best[0]} "
              f"{best[3] / best[1] / 1e6:.0f} GB/s", flush=True)
        G.set_staging(lev, which, 0)
