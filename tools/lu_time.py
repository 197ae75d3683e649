"""Time the config-1 batched LU (refactor) and one solve pass.
Usage: python tools/lu_time.py [n54 n59 reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_13201_b200 import fsigpu  # noqa: E402

n54 = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
n59 = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
B = fsigpu.DenseBlocks.generate_dominant(n54, n59, 20240901)
s = torch.cuda.Stream()
for _ in range(2):
    B.refactor(s.cuda_stream)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    B.refactor(s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
flops = n54 * 2.0 / 3.0 * 54 ** 3 + n59 * 2.0 / 3.0 * 59 ** 3
best = min(ts)
print(f"lu_ms {best:.3f} (all {[round(t, 3) for t in ts]}) TFLOP/s {flops / best / 1e9:.2f} "
      f"GB/s {(2 * B.factor_bytes + B.total_rows * 8) / best / 1e6:.0f}")
