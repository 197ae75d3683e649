"""Config-2 solve goldens from the UNMODIFIED reference (test infrastructure).

Runs the reference exporter (oracle/_ref/fsi_ref_harness, the reference's
own gmres on the additive FS hierarchy) on a config-2 case for
a bounded number of iterations and keeps only what a parity test needs
(a few KB): the recurrence history, iteration count, convergence flag, true
final residual, a strided sample of the iterate, and checksums of the
system so the test can tell that the fixture exported on the GPU box is the
same system. The operators themselves are re-exported on the box by the
same binary (tests/conftest.py), they are too large to commit.

usage: python oracle/make_cfg2_golden.py cfg2l4 [--max-iters 330] [--from EXPORT.fsix]
"""
from __future__ import annotations

import argparse
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_13201_b200 import fsix  # noqa: E402

STRIDE = 997


def system_checksums(a):
    """Order-sensitive checksums of the fine operator, RHS and scaling."""
    L = int(a["levels"][0])
    top = f"L{L - 1}"
    val = a[top + "/A/val"]
    w = np.arange(1, val.size + 1, dtype=np.float64) % 1009
    return np.array([float(a[top + "/A/rows"][0]), float(val.size), float(np.sum(val * w)),
                     float(np.sum(a["b"])), float(np.linalg.norm(a["b"])), float(np.sum(a["frame_scale"]))])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case", choices=["cfg2l4", "cfg2"])
    ap.add_argument("--max-iters", type=int, default=330)
    ap.add_argument("--from", dest="src", default=None, help="an existing export of the case")
    args = ap.parse_args()
    src = args.src
    if src is None:
        exe = os.path.join(ROOT, "oracle", "_ref", "fsi_ref_harness")
        src = os.path.join(tempfile.mkdtemp(), args.case + ".fsix")
        subprocess.run([exe, "export", args.case, src, "--no-mult", "--max-iters", str(args.max_iters)], check=True)
    a = fsix.load(src)
    out = {k: a[k] for k in ["gmres_add/history", "gmres_add/iterations", "gmres_add/converged",
                             "gmres_add/m_applies", "gmres_add/true_residual", "gmres/rel_tol"]}
    x = a["gmres_add/x"]
    out["gmres_add/x_sample"] = np.ascontiguousarray(x[::STRIDE])
    out["gmres_add/x_norm"] = np.array([np.linalg.norm(x)])
    out["x_sample_stride"] = np.array([STRIDE], np.int32)
    out["system_checksums"] = system_checksums(a)
    dst = os.path.join(ROOT, "tests", "golden", args.case + "_gmres.fsix")
    fsix.save(dst, out)
    print(f"{dst}: {int(out['gmres_add/iterations'][0])} its, converged {int(out['gmres_add/converged'][0])}, "
          f"{os.path.getsize(dst)} bytes")


if __name__ == "__main__":
    main()
