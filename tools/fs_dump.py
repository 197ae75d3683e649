"""Dump FS-apply and V-cycle outputs of the loaded build on config 0 (bitwise
comparison of two builds: FSIGPU_LIB=... python tools/fs_dump.py out.npz)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_13201_b200 import fsigpu  # noqa: E402
from paper_1909_13201_b200.problem import load_case  # noqa: E402

fsigpu.init(0)
P = load_case(os.path.join(ROOT, "data", "cfg0.fsix"), "cfg0")
G = fsigpu.GmgPreconditioner(P.levels)
r = np.random.default_rng(1).uniform(-1, 1, P.n)
out = {"fs": G.fs_apply(len(P.levels) - 1, r), "fs1": G.fs_apply(1, r[:P.levels[1].n]), "v": G.apply(r)}
np.savez(sys.argv[1], **out)
