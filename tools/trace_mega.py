"""Per-phase durations of the persistent kernel for the first Arnoldi steps."""
import ctypes as C
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_1909_13201_b200 import fsigpu
from paper_1909_13201_b200.problem import load_case
fsigpu.init(0)
L = fsigpu.lib()
L.fsigpu_debug_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int]
L.fsigpu_debug_trace.restype = C.c_int
P = load_case(os.path.join(ROOT, "data", "cfg0.fsix"))
G = fsigpu.GmgPreconditioner(P.levels)
S = fsigpu.GmresSolver(G, P.frame_scale, 30)
cfg = fsigpu.KrylovConfig(restart=30, max_iters=3, rel_tol=1e-10, abs_tol=1e-300)
S.solve(P.b, cfg)
buf = np.zeros(256, np.uint64)
L.fsigpu_debug_trace(S.h, buf.ctypes.data, 256, 1)
S.solve(P.b, cfg)
n = L.fsigpu_debug_trace(S.h, buf.ctypes.data, 256, 1)
t = buf[:n].astype(np.int64)
d = np.diff(t) / 1000.0
names = (["resid0", "norm0", "v0"] +
         (["L2 blk", "L2 comb", "L2 resid", "L2 restr", "L1 blk", "L1 comb", "L1 resid", "L1 restr", "coarse",
           "L1 prol", "L1 resid", "L1 blk", "L1 comb", "L2 prol", "L2 resid", "L2 blk", "L2 comb",
           "outer spmv", "dots", "upd+dots", "upd+norm", "normalize"]) * 3)
for i, x in enumerate(d):
    print(f"{i:3d} {names[i+1] if i+1 < len(names) else '?':12s} {x:8.2f} us")
print("total us", (t[-1] - t[0]) / 1000.0, "phases", n)
