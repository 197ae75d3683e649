"""A/B timing of config-1 block kernels under environment settings.
Usage: python tools/env_ab.py 'NAME=..,NAME2=..' 'NAME=..' ...   (each arg one variant;
'-' = defaults). Prints LU ms and mean batched-solve ms (100 solves)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, torch
sys.path.insert(0, ROOT)
from paper_1909_13201_b200 import fsigpu
B = fsigpu.DenseBlocks.generate_dominant(262144, 131072, 20240901)
s = torch.cuda.Stream()
rhs = torch.empty(B.total_rows, dtype=torch.float64, device="cuda")
x = torch.empty_like(rhs)
B.generate_rhs(7, rhs.data_ptr())
def t(fn, n):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(s)
    for _ in range(n): fn()
    e1.record(s); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
for _ in range(2): B.refactor(s.cuda_stream)
lu = min(t(lambda: B.refactor(s.cuda_stream), 1) for _ in range(3))
for _ in range(3): B.solve_dev(rhs.data_ptr(), x.data_ptr(), s.cuda_stream)
sv = t(lambda: B.solve_dev(rhs.data_ptr(), x.data_ptr(), s.cuda_stream), 100)
xh = x[:54].cpu().numpy()
sys.path.insert(0, ROOT + "/oracle")
import oracle as O
lu_, piv = O.dense_factor(B.matrix(0, 54))
import numpy as np
xo = O.dense_solve(lu_, piv, rhs[:54].cpu().numpy())
err = float(np.linalg.norm(xh - xo) / np.linalg.norm(xo))
fb = B.factor_bytes
print(json.dumps({"lu_ms": lu, "solve_ms": sv, "solve_GBps": (fb + B.total_rows * 20) / sv / 1e6, "err0": err}))
'''

if __name__ == "__main__":
    code = CHILD.replace("ROOT", repr(ROOT))
    for v in sys.argv[1:] or ["-"]:
        env = dict(os.environ)
        if v != "-":
            for kv in v.split(","):
                k, val = kv.split("=")
                env[k] = val
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-1500:]
        print(v, line, flush=True)
