import ctypes as C
import os, sys, time, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_1909_13201_b200 import fsigpu
from paper_1909_13201_b200.problem import load_case


def one(limit):
    fsigpu.init(0)
    L = fsigpu.lib()
    L.fsigpu_debug_phase_limit.argtypes = [C.c_void_p, C.c_uint]
    P = load_case(os.path.join(ROOT, "tests", "golden", "chan.fsix"))
    G = fsigpu.GmgPreconditioner(P.levels)
    S = fsigpu.GmresSolver(G, P.frame_scale, 30)
    fsigpu._check(L.fsigpu_debug_phase_limit(S.h, limit))
    cfg = fsigpu.KrylovConfig(restart=30, max_iters=1, rel_tol=1e-8, abs_tol=1e-300)
    t = time.time()
    try:
        r = S.solve(P.b, cfg)
        print("limit", limit, "returned its", r.iterations, round(time.time() - t, 3), flush=True)
    except Exception as e:
        print("limit", limit, "error", e, round(time.time() - t, 3), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        one(int(sys.argv[1]))
        sys.exit(0)
    fsigpu.init(0)
    L = fsigpu.lib()
    L.fsigpu_debug_barrier.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
    for kind in [0, 1, 2]:
        for grid in [148, 296]:
            ms = C.c_double()
            rc = L.fsigpu_debug_barrier(grid, 2000, kind, C.byref(ms))
            print("barrier kind", kind, "grid", grid, "rc", rc, L.fsigpu_last_error(), "us/barrier", ms.value * 1000 / 2000, flush=True)
    for limit in [2, 40, 0]:
        try:
            out = subprocess.run([sys.executable, __file__, str(limit)], capture_output=True, text=True, timeout=25)
            print(out.stdout.strip()[-300:], out.stderr.strip()[-300:], flush=True)
        except subprocess.TimeoutExpired:
            print("limit", limit, "TIMEOUT", flush=True)
