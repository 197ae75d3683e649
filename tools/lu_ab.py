"""A/B timing of the config-1 batched LU (262,144 x m=54 + 131,072 x m=59):
register-row kernel (default) vs the shared-memory CTA kernel
(FSIGPU_LU_SMEM=1). Usage: python tools/lu_ab.py [n54 n59]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, torch
sys.path.insert(0, ROOT)
from paper_1909_13201_b200 import fsigpu
n54, n59 = N54, N59
B = fsigpu.DenseBlocks.generate_dominant(n54, n59, 20240901)
s = torch.cuda.Stream()
for _ in range(2):
    B.refactor(s.cuda_stream)
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(s); B.refactor(s.cuda_stream); e1.record(s); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
flops = n54 * 2 / 3 * 54 ** 3 + n59 * 2 / 3 * 59 ** 3
ms = min(ts)
print(json.dumps({"lu_ms": ms, "all_ms": ts, "TFLOPs": flops / ms / 1e9, "GBps": 2 * B.factor_bytes / ms / 1e6}))
'''

if __name__ == "__main__":
    n54 = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
    n59 = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
    code = CHILD.replace("ROOT", repr(ROOT)).replace("N54", str(n54)).replace("N59", str(n59))
    for var, env in [("register", "0"), ("smem", "1")]:
        out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, FSIGPU_LU_SMEM=env),
                             capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-2000:]
        print(var, line, flush=True)
