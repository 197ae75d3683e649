"""One config-1-style batched LU (for ncu captures of the LU kernels).
Usage: python tools/lu_only.py [n54 n59]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_13201_b200 import fsigpu  # noqa: E402

n54 = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
n59 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
B = fsigpu.DenseBlocks.generate_dominant(n54, n59, 20240901)
torch.cuda.synchronize()
print("factored", B.total_rows, "rows")
if len(sys.argv) > 3 and sys.argv[3] == "solve":
    rhs = torch.empty(B.total_rows, dtype=torch.float64, device="cuda")
    x = torch.empty_like(rhs)
    B.generate_rhs(7, rhs.data_ptr())
    s = torch.cuda.Stream()
    for _ in range(3):
        B.solve_dev(rhs.data_ptr(), x.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    print("solved")
