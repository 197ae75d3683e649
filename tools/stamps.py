"""In-graph kernel durations of one solve (device-clock stamps), config 0 by default.
Usage: [FSI_DATA=...] python tools/stamps.py [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1909_13201_b200 import fsigpu  # noqa: E402
from paper_1909_13201_b200.problem import load_case  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
fsigpu.init(0)
P = load_case(os.environ.get("FSI_DATA", os.path.join(ROOT, "data", "cfg0.fsix")), "case")
G = fsigpu.GmgPreconditioner(P.levels)
S = fsigpu.GmresSolver(G, P.frame_scale, restart=30)
cfg = fsigpu.KrylovConfig(restart=30, max_iters=int(os.environ.get("FSI_MAXIT", "2000")), rel_tol=1e-10, abs_tol=1e-300)
top = len(P.levels) - 1
b = torch.from_numpy(P.b).cuda()
x = torch.zeros(P.b.shape[0], dtype=torch.float64, device="cuda")
stream = torch.cuda.ExternalStream(G.stream())
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for _ in range(2):
    x.zero_()
    S.solve_dev(b.data_ptr(), x.data_ptr(), cfg)
ts = []
for _ in range(reps):
    flush.fill_(1.0)
    x.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    r = S.solve_dev(b.data_ptr(), x.data_ptr(), cfg)
    e1.record(stream)
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"plain: {min(ts):.3f} ms per solve, {r.iterations} its, {1000 * min(ts) / r.iterations:.1f} us per step")
fsigpu.Stamps.enable(True)
x.zero_()
S.solve_dev(b.data_ptr(), x.data_ptr(), cfg)
fsigpu.Stamps.enable(True)
flush.fill_(1.0)
x.zero_()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
r = S.solve_dev(b.data_ptr(), x.data_ptr(), cfg)
e1.record(stream)
e1.synchronize()
names = {}
for lvl in range(top, -1, -1):
    names[f"fs_smoother@L{lvl}"] = ("block_solve", lvl, 0)
    names[f"residual@L{lvl}"] = ("spmv", lvl, 0)
    names[f"restrict@L{lvl}"] = ("transfer", lvl, 0)
    names[f"prolong_resid@L{lvl}"] = ("transfer", lvl, 1)
names["coarse@L0"] = ("coarse", 0, 0)
names["outer SpMV (split A)"] = ("spmv", -1, 0)
names["arnoldi A"] = ("arnoldi", -1, 0)
names["arnoldi B"] = ("arnoldi", -1, 1)
names["arnoldi C"] = ("arnoldi", -1, 2)
tot = 0.0
for nm, (c, l, s) in names.items():
    v = fsigpu.Stamps.read(c, l, s)
    if v["launches"]:
        print(f"{nm:22s} {v['us'] / v['launches']:8.2f} us x {v['launches'] / r.iterations:.0f} per step")
        tot += v["us"]
print(f"stamped {tot / r.iterations:.1f} us per step; solve with stamps {1000 * e0.elapsed_time(e1) / r.iterations:.1f} us per step")
fsigpu.Stamps.enable(False)
