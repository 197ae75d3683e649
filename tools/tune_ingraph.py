"""Sweep SpMV launch shapes (lanes per row x batch depth) per level and matrix with the
kernel's IN-GRAPH duration (device-clock stamps inside the captured restart-cycle graph of a
real solve) as the objective. Usage: [FSI_DATA=...] [FSI_MAXIT=..] python tools/tune_ingraph.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1909_13201_b200 import fsigpu  # noqa: E402
from paper_1909_13201_b200.problem import load_case  # noqa: E402

fsigpu.init(0)
P = load_case(os.environ.get("FSI_DATA", os.path.join(ROOT, "data", "cfg0.fsix")), "case")
G = fsigpu.GmgPreconditioner(P.levels)
S = fsigpu.GmresSolver(G, P.frame_scale, restart=30)
cfg = fsigpu.KrylovConfig(restart=30, max_iters=int(os.environ.get("FSI_MAXIT", "60")), rel_tol=1e-10, abs_tol=1e-300)
top = len(P.levels) - 1
b = torch.from_numpy(P.b).cuda()
x = torch.zeros(P.b.shape[0], dtype=torch.float64, device="cuda")
KEY = {"A": ("spmv", 0), "FS": ("block_solve", 0), "AP": ("transfer", 1), "R": ("transfer", 0)}


def measure(level, which):
    cls, sub = KEY[which]
    lv = level  # R of level l (to l - 1) is stored and launched under level l
    fsigpu.Stamps.enable(True)
    x.zero_()
    S.solve_dev(b.data_ptr(), x.data_ptr(), cfg)  # re-capture
    fsigpu.Stamps.enable(True)
    best = None
    for _ in range(3):
        x.zero_()
        S.solve_dev(b.data_ptr(), x.data_ptr(), cfg)
    v = fsigpu.Stamps.read(cls, lv, sub)
    return v["us"] / max(v["launches"], 1)


for lev in range(top, 0, -1):
    for which in ["FS", "A", "AP", "R"]:
        measure(lev, which)  # warm-up: the first measurement after a re-capture reads high
        base = measure(lev, which)
        res = []
        for lpr in [2, 4, 8, 16, 32]:
            for u in [4, 8, 22, 24]:
                try:
                    G.set_launch(lev, which, lpr, u)
                except Exception:
                    continue
                res.append((measure(lev, which), lpr, u))
        res.sort()
        print(f"L{lev} {which:3s} default {base:6.2f} us | best " +
              ", ".join(f"lpr={l} u={u}: {t:.2f}" for t, l, u in res[:4]), flush=True)
        G.set_launch(lev, which, res[0][1], res[0][2])
fsigpu.Stamps.enable(False)
