"""Batched LU of large blocks (the config-4 regime, m ~ 500-780, pure-DD
Vanka patches): time of the refactor for `count` random diagonally dominant
blocks of size m, and a sampled parity check against the oracle.
Usage: python tools/lu_large.py m count"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_1909_13201_b200 import fsigpu  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 500
count = int(sys.argv[2]) if len(sys.argv) > 2 else 148
rng = np.random.default_rng(5)
mats = []
for _ in range(count):
    a = rng.uniform(-1, 1, (m, m))
    a[np.diag_indices(m)] += np.abs(a).sum(axis=1)
    mats.append(a)
t0 = time.time()
B = fsigpu.DenseBlocks.from_dense(mats)
first = time.time() - t0
s = torch.cuda.Stream()
B.refactor(s.cuda_stream)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
B.refactor(s.cuda_stream)
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
flops = count * 2.0 / 3.0 * m ** 3
import oracle as O  # noqa: E402
rhs = rng.uniform(-1, 1, count * m)
x = B.solve(rhs)
lu, piv = O.dense_factor(mats[0])
xo = O.dense_solve(lu, piv, rhs[:m])
print(json.dumps({"m": m, "blocks": count, "lu_ms": ms, "TFLOPs": flops / ms / 1e9,
                  "GBps_2x_matrix": 2 * 8.0 * count * m * m / ms / 1e6,
                  "rel_err_block0": float(np.linalg.norm(x[:m] - xo) / np.linalg.norm(xo)), "first_s": first}))
