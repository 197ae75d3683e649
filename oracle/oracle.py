"""ctypes binding of the C restatement oracle (oracle/fsi_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / reference legs of bench.py, always as the checker or the
reported CPU baseline — never on the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "liboracle.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"oracle not built: {LIB_PATH} (run `make -C oracle oracle`)")
        L = C.CDLL(LIB_PATH)
        vp, ip = C.c_void_p, C.c_int
        L.orc_csr_spmv.argtypes = [ip, vp, vp, vp, vp, vp]
        L.orc_dense_factor.argtypes = [ip, vp, vp]
        L.orc_dense_factor.restype = ip
        L.orc_dense_solve.argtypes = [ip, vp, vp, vp, vp]
        L.orc_extract_block.argtypes = [vp, vp, vp, ip, vp, vp]
        L.orc_gmg_create.argtypes = [ip, vp, C.c_double, ip, ip, C.POINTER(ip), C.POINTER(ip)]
        L.orc_gmg_create.restype = vp
        L.orc_gmg_destroy.argtypes = [vp]
        L.orc_gmg_set_cycle.argtypes = [vp, C.c_char]
        L.orc_fs_apply.argtypes = [vp, ip, vp, vp]
        L.orc_gmg_apply.argtypes = [vp, vp, vp]
        L.orc_coarse_solve.argtypes = [vp, vp, vp]
        L.orc_gmres.argtypes = [vp, vp, vp, ip, ip, C.c_double, C.c_double, vp, vp,
                                C.POINTER(ip), C.POINTER(ip), C.POINTER(ip), C.POINTER(ip),
                                C.POINTER(C.c_longlong)]
        L.orc_gmres.restype = ip
        L.orc_fgmres.argtypes = L.orc_gmres.argtypes
        L.orc_fgmres.restype = ip
        L.orc_gmg_set_smoother.argtypes = [vp, ip]
        L.orc_gmg_set_fs_mode.argtypes = [vp, ip]
        L.orc_gmg_colours.argtypes = [vp, ip, ip]
        L.orc_gmg_colours.restype = ip
        _lib = L
    return _lib


def _d(a):
    return np.ascontiguousarray(a, np.float64)


def spmv(A, x):
    x = _d(x)
    y = np.empty(A.rows)
    lib().orc_csr_spmv(A.rows, A.ptr.ctypes.data, A.idx.ctypes.data, A.val.ctypes.data,
                       x.ctypes.data, y.ctypes.data)
    return y


def dense_factor(a):
    """DenseFactorization ctor: returns (lu row-major, piv) or raises."""
    m = a.shape[0]
    lu = np.ascontiguousarray(a, np.float64).copy()
    piv = np.zeros(m, np.int32)
    if lib().orc_dense_factor(m, lu.ctypes.data, piv.ctypes.data):
        raise ZeroDivisionError("singular block")
    return lu, piv


def dense_solve(lu, piv, b):
    m = lu.shape[0]
    b = _d(b)
    x = np.empty(m)
    lib().orc_dense_solve(m, lu.ctypes.data, piv.ctypes.data, b.ctypes.data, x.ctypes.data)
    return x


def extract_block(A, dofs):
    dofs = np.ascontiguousarray(dofs, np.int32)
    m = len(dofs)
    d = np.empty((m, m))
    lib().orc_extract_block(A.ptr.ctypes.data, A.idx.ctypes.data, A.val.ctypes.data, m,
                            dofs.ctypes.data, d.ctypes.data)
    return d


class OracleGmg:
    """GmgPreconditioner with FS smoothers (CPU restatement). fs: "additive"
    (default), "multicolour" (multiplicative in the multicolour
    block order the GPU runs) or "multiplicative" (the shipped
    FsPreconditioner::apply, blocks in the reference's order)."""

    SMOOTHERS = {"richardson": 0, "gmres1": 1}
    FS_MODES = {"additive": 0, "multicolour": 1, "multiplicative": 2}

    def __init__(self, levels: List, omega=0.7, pre=1, post=1, cycle="v", smoother="richardson",
                 fs="additive"):
        from paper_1909_13201_b200.problem import level_descs
        self.levels = levels
        self._descs = level_descs(levels)
        el, eb = C.c_int(), C.c_int()
        h = lib().orc_gmg_create(len(levels), C.addressof(self._descs), omega, pre, post,
                                 C.byref(el), C.byref(eb))
        if not h:
            raise ZeroDivisionError(f"singular block: level {el.value} block {eb.value}")
        self.h = h
        lib().orc_gmg_set_cycle(h, cycle.encode()[:1])
        lib().orc_gmg_set_smoother(h, self.SMOOTHERS[smoother])
        lib().orc_gmg_set_fs_mode(h, self.FS_MODES[fs])

    def colours(self, level, group):
        """Colour count of the AS1 (group 1) or AS2 (group 2) blocks of a level."""
        return lib().orc_gmg_colours(self.h, level, group)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_gmg_destroy(self.h)
            self.h = None

    def fs_apply(self, level, r):
        r = _d(r)
        z = np.empty_like(r)
        lib().orc_fs_apply(self.h, level, r.ctypes.data, z.ctypes.data)
        return z

    def apply(self, r):
        r = _d(r)
        z = np.empty_like(r)
        lib().orc_gmg_apply(self.h, r.ctypes.data, z.ctypes.data)
        return z

    def coarse_solve(self, b):
        b = _d(b)
        x = np.empty_like(b)
        lib().orc_coarse_solve(self.h, b.ctypes.data, x.ctypes.data)
        return x

    def gmres(self, frame_scale, b, restart=30, max_iters=2000, rel_tol=1e-10, abs_tol=1e-300,
              flexible=False):
        n = len(b)
        b, fsc = _d(b), _d(frame_scale)
        x = np.empty(n)
        hist = np.empty(max_iters + 2)
        nh, it, cv, bk = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        ma = C.c_longlong()
        fn = lib().orc_fgmres if flexible else lib().orc_gmres
        rc = fn(self.h, fsc.ctypes.data, b.ctypes.data, restart, max_iters, rel_tol,
                             abs_tol, x.ctypes.data, hist.ctypes.data, C.byref(nh), C.byref(it),
                             C.byref(cv), C.byref(bk), C.byref(ma))
        if rc:
            raise ValueError("gmres: invalid config")
        return dict(x=x, history=hist[:nh.value].copy(), iterations=it.value,
                    converged=bool(cv.value), breakdown=bool(bk.value), m_applies=ma.value)
