"""A/B timing of config-0 solves under library switches (device time, CUDA events)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_1909_13201_b200 import fsigpu
from paper_1909_13201_b200.problem import load_case

fsigpu.init(0)
P = load_case(os.path.join(ROOT, "data", "cfg0.fsix"))
cfg = fsigpu.KrylovConfig(restart=30, max_iters=2000, rel_tol=1e-10, abs_tol=1e-300)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")


def run(tag, persist=True, mode=fsigpu.MODE_INVERSE, mega=False, reps=5, pdl=True):
    fsigpu.set_pdl(pdl)
    fsigpu.set_l2_persist(persist)
    fsigpu.set_block_mode(mode)
    G = fsigpu.GmgPreconditioner(P.levels)
    S = fsigpu.GmresSolver(G, P.frame_scale, 30)
    if mega:
        S.set_persistent(True)
    st = torch.cuda.ExternalStream(G.stream())
    b = torch.from_numpy(P.b).cuda()
    x = torch.zeros_like(b)
    ts = []
    for k in range(reps + 2):
        flush.fill_(1.0)
        x.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        r = S.solve_dev(b.data_ptr(), x.data_ptr(), cfg)
        e1.record(st)
        e1.synchronize()
        if k >= 2:
            ts.append(e0.elapsed_time(e1))
    print(f"{tag:28s} its={r.iterations} solve_ms median={np.median(ts):.3f} min={min(ts):.3f} persist={G.persist_bytes()}", flush=True)
    fsigpu.set_l2_persist(False)
    fsigpu.set_block_mode(fsigpu.MODE_ASSEMBLED)


if __name__ == "__main__":
    run("assembled, no PDL", False, fsigpu.MODE_ASSEMBLED, pdl=False)
    run("assembled", False, fsigpu.MODE_ASSEMBLED)
    run("inverse", False, fsigpu.MODE_INVERSE)
    run("LU", False, fsigpu.MODE_LU)
    run("inverse, mega", False, fsigpu.MODE_INVERSE, mega=True)
    run("assembled, persist", True, fsigpu.MODE_ASSEMBLED)
