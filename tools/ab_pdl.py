"""A/B of programmatic dependent launch on the config-0 solve (and config 2
when data_cfg2/cfg2.fsix exists): device time per FGMRES(30) solve, L2
flushed between solves, PDL off vs on, interleaved rounds.
Usage: python tools/ab_pdl.py [cfg0|cfg2] [rounds]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_13201_b200 import fsigpu  # noqa: E402
from paper_1909_13201_b200.problem import load_case  # noqa: E402


def main():
    case = sys.argv[1] if len(sys.argv) > 1 else "cfg0"
    rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    path = os.path.join(ROOT, "data", "cfg0.fsix") if case == "cfg0" else os.path.join(ROOT, "data_cfg2", case + ".fsix")
    P = load_case(path)
    fsigpu.init(0)
    max_iters = 2000 if case == "cfg0" else 60
    cfg = fsigpu.KrylovConfig(restart=30, max_iters=max_iters, rel_tol=1e-10, abs_tol=1e-300)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    b = torch.from_numpy(P.b).cuda()
    x = torch.zeros(P.n, dtype=torch.float64, device="cuda")
    solvers = {}
    for pdl in (0, 1):
        fsigpu.set_pdl(bool(pdl))
        G = fsigpu.GmgPreconditioner(P.levels)
        S = fsigpu.GmresSolver(G, P.frame_scale, 30)
        for _ in range(3):
            S.solve_dev(b.data_ptr(), x.data_ptr(), cfg)  # captures the graph with this PDL setting
        solvers[pdl] = (G, S)
    res = {0: [], 1: []}
    for r in range(rounds):
        for pdl in (0, 1):
            fsigpu.set_pdl(bool(pdl))
            G, S = solvers[pdl]
            st = torch.cuda.ExternalStream(G.stream())
            for _ in range(10):
                flush.fill_(1.0)
                x.zero_()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                out = S.solve_dev(b.data_ptr(), x.data_ptr(), cfg)
                e1.record(st)
                e1.synchronize()
                res[pdl].append(e0.elapsed_time(e1))
    for pdl in (0, 1):
        v = np.array(res[pdl])
        print(f"{case} pdl={pdl}: median {np.median(v):.3f} ms  min {v.min():.3f}  its {out.iterations}")


if __name__ == "__main__":
    main()
