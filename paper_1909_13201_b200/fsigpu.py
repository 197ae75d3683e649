"""Host-side mirror of the reference solve-layer interface over libfsigpu.

Same names, argument meaning and error behaviour as the reference C++
classes this path replaces (citations into /root/reference/proj):

=====================  =============================================  =====================
this module            reference                                      C ABI (include/fsigpu.h)
=====================  =============================================  =====================
SparseMatrix.multiply  SparseMatrix::multiply  src/sparse.cpp:70-76      fsigpu_csr_multiply
DenseBlocks            DenseFactorization      src/dense.cpp:31-86       fsigpu_blocks_*
DenseBlocks.from_csr   factor_principal_block  src/precond.cpp:13-21     fsigpu_blocks_factor_csr
GmgPreconditioner      GmgPreconditioner       src/gmg.cpp:178-246       fsigpu_gmg_*
  .fs_apply            FsPreconditioner::apply src/precond.cpp:271-303   fsigpu_fs_apply
                       (additive Schwarz)
gmres                  gmres                   src/krylov.cpp:20-126     fsigpu_gmres_*
KrylovConfig           KrylovConfig            include/fsi/krylov.hpp:42-47
GmresResult            GmresResult             include/fsi/krylov.hpp:49-55
SingularBlockError     SingularBlockError      include/fsi/errors.hpp:12-20
=====================  =============================================  =====================

There is no CPU fallback: importing works without a GPU (so the CPU test
tier can check the ABI), but every compute call goes through the CUDA
library and raises if it is missing or no device is present.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from .problem import BlockSets, Csr, Level, level_descs, mesh_desc

_HERE = os.path.dirname(os.path.abspath(__file__))
# FSIGPU_LIB: an alternative in-tree build of the same library (A/B timing
# of two builds, tools/ab_build.sh); default the package's own libfsigpu.so
LIB_PATH = os.environ.get("FSIGPU_LIB") or os.path.join(_HERE, "libfsigpu.so")

FSIGPU_OK, FSIGPU_ERR_INVALID, FSIGPU_ERR_SINGULAR, FSIGPU_ERR_CUDA = 0, 1, 2, 3
KERNEL_CLASSES = ["block_solve", "spmv", "transfer", "combine", "coarse", "arnoldi"]


class SingularBlockError(RuntimeError):
    """Zero or near-zero pivot in a block factorization (errors.hpp:12-20)."""

    def __init__(self, label: str):
        super().__init__("singular block: " + label)
        self.label = label


class SolverError(RuntimeError):
    pass


class GmresResultC(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("breakdown", C.c_int),
                ("n_history", C.c_int), ("m_applies", C.c_longlong), ("true_residual", C.c_double)]


_lib = None
_initialised = False


def lib():
    """Load libfsigpu.so (raises if it was not built: no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libfsigpu.so missing at {LIB_PATH}: run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        vp, ip, ll, d = C.c_void_p, C.c_int, C.c_longlong, C.c_double
        sig = {
            "fsigpu_last_error": ([], C.c_char_p),
            "fsigpu_last_singular_block": ([], ip),
            "fsigpu_last_singular_level": ([], ip),
            "fsigpu_init": ([ip], ip),
            "fsigpu_version": ([], ip),
            "fsigpu_launch_count": ([], ll),
            "fsigpu_set_block_mode": ([ip], ip),
            "fsigpu_set_pdl": ([ip], ip),
            "fsigpu_gmg_stream": ([vp], vp),
            "fsigpu_csr_create": ([ip, ip, vp, vp, vp, C.POINTER(vp)], ip),
            "fsigpu_csr_multiply": ([vp, vp, vp], ip),
            "fsigpu_csr_multiply_dev": ([vp, vp, vp, vp], ip),
            "fsigpu_csr_time": ([vp, ip, C.POINTER(d)], ip),
            "fsigpu_csr_destroy": ([vp], None),
            "fsigpu_blocks_factor_csr": ([vp, ip, vp, vp, C.POINTER(vp)], ip),
            "fsigpu_blocks_factor_dense": ([ip, vp, vp, C.POINTER(vp)], ip),
            "fsigpu_blocks_generate_dominant": ([ll, ll, C.c_ulonglong, C.POINTER(vp)], ip),
            "fsigpu_blocks_generate_rhs": ([vp, C.c_ulonglong, vp], ip),
            "fsigpu_blocks_copy_matrix": ([vp, ll, vp], ip),
            "fsigpu_blocks_count": ([vp], ll),
            "fsigpu_blocks_total_rows": ([vp], ll),
            "fsigpu_blocks_factor_bytes": ([vp], ll),
            "fsigpu_blocks_solve": ([vp, vp, vp], ip),
            "fsigpu_blocks_solve_dev": ([vp, vp, vp, vp], ip),
            "fsigpu_blocks_refactor": ([vp, vp], ip),
            "fsigpu_blocks_get_lu": ([vp, vp, vp], ip),
            "fsigpu_blocks_destroy": ([vp], None),
            "fsigpu_gmg_create": ([ip, vp, d, ip, ip, C.c_char, C.POINTER(vp)], ip),
            "fsigpu_gmg_create_ex": ([ip, vp, d, ip, ip, C.c_char, ip, C.POINTER(vp)], ip),
            "fsigpu_gmg_size": ([vp], ip),
            "fsigpu_gmg_apply": ([vp, vp, vp], ip),
            "fsigpu_gmg_apply_dev": ([vp, vp, vp, vp], ip),
            "fsigpu_fs_apply": ([vp, ip, vp, vp], ip),
            "fsigpu_coarse_solve": ([vp, vp, vp], ip),
            "fsigpu_gmg_destroy": ([vp], None),
            "fsigpu_gmg_set_launch": ([vp, ip, ip, ip, ip], ip),
            "fsigpu_gmg_set_smoother": ([vp, ip], ip),
            "fsigpu_gmg_time_kernel": ([vp, ip, ip, ip, ip, C.POINTER(d), C.POINTER(d)], ip),
            "fsigpu_gmres_create": ([vp, vp, ip, C.POINTER(vp)], ip),
            "fsigpu_gmres_solve": ([vp, vp, vp, vp, ip, d, d, vp, C.POINTER(GmresResultC)], ip),
            "fsigpu_gmres_solve_dev": ([vp, vp, vp, ip, d, d, vp, C.POINTER(GmresResultC)], ip),
            "fsigpu_gmres_set_graphs": ([vp, ip], ip),
            "fsigpu_gmres_destroy": ([vp], None),
            "fsigpu_fs_sets_build": ([vp, vp, ip, ip, ip, C.POINTER(vp)], ip),
            "fsigpu_vanka_sets_build": ([ip, vp, ip, C.POINTER(vp)], ip),
            "fsigpu_sets_counts": ([vp, C.POINTER(ip), C.POINTER(ip), C.POINTER(ip), C.POINTER(ip),
                                    C.POINTER(ip)], ip),
            "fsigpu_sets_copy": ([vp, vp, vp, vp, vp, vp], ip),
            "fsigpu_sets_label": ([vp, ip], C.c_char_p),
            "fsigpu_sets_destroy": ([vp], None),
            "fsigpu_profile_enable": ([ip], ip),
            "fsigpu_profile_read": ([vp, vp, vp], ip),
            "fsigpu_profile_read_level": ([ip, ip, vp, vp, vp], ip),
            "fsigpu_profile_reset": ([], ip),
            "fsigpu_stamps_enable": ([ip], ip),
            "fsigpu_stamps_read": ([ip, ip, ip, vp, vp], ip),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _check(rc: int, labels: Optional[Sequence[str]] = None):
    if rc == FSIGPU_OK:
        return
    L = lib()
    msg = L.fsigpu_last_error().decode()
    if rc == FSIGPU_ERR_SINGULAR:
        b = L.fsigpu_last_singular_block()
        if labels is not None and 0 <= b < len(labels):
            raise SingularBlockError(labels[b])
        raise SingularBlockError(msg.replace("singular block: ", ""))
    if rc == FSIGPU_ERR_INVALID:
        raise ValueError(msg)
    raise SolverError(msg)


def init(device: int = 0):
    global _initialised
    if not _initialised:
        _check(lib().fsigpu_init(device))
        _initialised = True


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


class SparseMatrix:
    """Device CSR matrix; ``multiply`` is SparseMatrix::multiply."""

    def __init__(self, a: Csr):
        init()
        self._keep = (_i32(a.ptr), _i32(a.idx), _f64(a.val))
        self.rows, self.cols = a.rows, a.cols
        h = C.c_void_p()
        _check(lib().fsigpu_csr_create(a.rows, a.cols, self._keep[0].ctypes.data,
                                       self._keep[1].ctypes.data, self._keep[2].ctypes.data, C.byref(h)))
        self.h = h

    def multiply(self, x) -> np.ndarray:
        x = _f64(x)
        if x.shape != (self.cols,):
            raise ValueError("spmv: dimension mismatch")
        y = np.empty(self.rows)
        _check(lib().fsigpu_csr_multiply(self.h, x.ctypes.data, y.ctypes.data))
        return y

    def time_spmv(self, reps: int = 100) -> float:
        ms = C.c_double()
        _check(lib().fsigpu_csr_time(self.h, reps, C.byref(ms)))
        return ms.value

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.fsigpu_csr_destroy(self.h)
            self.h = None


class DenseBlocks:
    """Batch of DenseFactorization objects living on the device."""

    def __init__(self, handle, labels: Optional[List[str]] = None, owner=None):
        self.h = handle
        self.labels = labels
        self._owner = owner
        L = lib()
        self.count = L.fsigpu_blocks_count(self.h)
        self.total_rows = L.fsigpu_blocks_total_rows(self.h)
        self.factor_bytes = L.fsigpu_blocks_factor_bytes(self.h)

    @staticmethod
    def from_dense(mats: Sequence[np.ndarray], labels: Optional[List[str]] = None) -> "DenseBlocks":
        init()
        sizes = _i32([m.shape[0] for m in mats])
        for m in mats:
            if m.ndim != 2 or m.shape[0] != m.shape[1]:
                raise ValueError("lu: matrix not square")
        flat = _f64(np.concatenate([np.ravel(m) for m in mats])) if len(mats) else np.zeros(1)
        h = C.c_void_p()
        _check(lib().fsigpu_blocks_factor_dense(len(mats), sizes.ctypes.data, flat.ctypes.data, C.byref(h)),
               labels)
        return DenseBlocks(h, labels)

    @staticmethod
    def from_csr(a: SparseMatrix, sets: Sequence[np.ndarray],
                 labels: Optional[List[str]] = None) -> "DenseBlocks":
        ptr = _i32(np.concatenate([[0], np.cumsum([len(s) for s in sets])]))
        idx = _i32(np.concatenate([np.asarray(s) for s in sets])) if len(sets) else np.zeros(1, np.int32)
        h = C.c_void_p()
        _check(lib().fsigpu_blocks_factor_csr(a.h, len(sets), ptr.ctypes.data, idx.ctypes.data, C.byref(h)),
               labels)
        return DenseBlocks(h, labels, owner=a)

    @staticmethod
    def generate_dominant(n54: int, n59: int, seed: int) -> "DenseBlocks":
        init()
        h = C.c_void_p()
        _check(lib().fsigpu_blocks_generate_dominant(n54, n59, seed, C.byref(h)))
        return DenseBlocks(h)

    def matrix(self, b: int, m: int) -> np.ndarray:
        out = np.empty((m, m))
        _check(lib().fsigpu_blocks_copy_matrix(self.h, b, out.ctypes.data))
        return out

    def solve(self, rhs) -> np.ndarray:
        rhs = _f64(rhs)
        if rhs.shape != (self.total_rows,):
            raise ValueError("lu solve: size mismatch")
        x = np.empty(self.total_rows)
        _check(lib().fsigpu_blocks_solve(self.h, rhs.ctypes.data, x.ctypes.data))
        return x

    def solve_dev(self, d_rhs: int, d_x: int, stream: int = 0):
        _check(lib().fsigpu_blocks_solve_dev(self.h, C.c_void_p(d_rhs), C.c_void_p(d_x), C.c_void_p(stream)))

    def generate_rhs(self, seed: int, d_rhs: int):
        _check(lib().fsigpu_blocks_generate_rhs(self.h, seed, C.c_void_p(d_rhs)))

    def refactor(self, stream: int = 0):
        _check(lib().fsigpu_blocks_refactor(self.h, C.c_void_p(stream)), self.labels)

    def lu(self, sizes: Sequence[int]):
        tot = int(sum(int(m) * int(m) for m in sizes))
        lu = np.empty(max(tot, 1))
        piv = np.empty(max(self.total_rows, 1), np.int32)
        _check(lib().fsigpu_blocks_get_lu(self.h, lu.ctypes.data, piv.ctypes.data))
        out, o, r = [], 0, 0
        for m in sizes:
            m = int(m)
            out.append((lu[o:o + m * m].reshape(m, m), piv[r:r + m]))
            o += m * m
            r += m
        return out

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.fsigpu_blocks_destroy(self.h)
            self.h = None


@dataclass
class CycleConfig:
    """gmg.hpp:54-58"""
    cycle: str = "v"
    pre: int = 1
    post: int = 1
    omega: float = 0.7
    # "richardson" (precond.cpp:305-317) or "gmres1" (minimal-residual step,
    # BASELINE configs[0]; non-linear, use under the flexible device solver)
    smoother: str = "richardson"
    # SchwarzMode of the FS blocks (include/fsi/precond.hpp): "additive"
    # (default) or "multiplicative" (the shipped
    # FsPreconditioner::apply, precond.cpp:271-303, blocks in multicolour order)
    schwarz: str = "additive"


class GmgPreconditioner:
    """GMG V/W/F cycle with FS smoothers on the device."""

    def __init__(self, levels: List[Level], cfg: CycleConfig = CycleConfig()):
        init()
        self.levels = levels
        self._descs = level_descs(levels)
        self.labels = []
        h = C.c_void_p()
        rc = lib().fsigpu_gmg_create_ex(len(levels), C.addressof(self._descs), cfg.omega, cfg.pre, cfg.post,
                                        cfg.cycle.encode()[:1], self.SCHWARZ[cfg.schwarz], C.byref(h))
        if rc == FSIGPU_ERR_SINGULAR:
            # the failing block's reference label (precond.cpp:182,224,265)
            b, lvl = lib().fsigpu_last_singular_block(), lib().fsigpu_last_singular_level()
            labels = levels[lvl].labels if 0 <= lvl < len(levels) else None
            if labels is not None and 0 <= b < len(labels):
                raise SingularBlockError(labels[b])
            msg = lib().fsigpu_last_error().decode()
            raise SingularBlockError(msg.replace("singular block: ", ""))
        _check(rc)
        self.h = h
        self.n = levels[-1].n
        if cfg.smoother != "richardson":
            self.set_smoother(cfg.smoother)

    SMOOTHERS = {"richardson": 0, "gmres1": 1}
    SCHWARZ = {"additive": 0, "multiplicative": 1}

    def set_smoother(self, kind: str):
        _check(lib().fsigpu_gmg_set_smoother(self.h, self.SMOOTHERS[kind]))

    def size(self) -> int:
        return self.n

    KERNELS = {"fs_smoother": 0, "residual": 1, "prolong_resid": 2, "restrict": 3, "coarse": 4}

    def time_kernel(self, which: str, level: int, reps: int = 20, cold: bool = True):
        """(ms per launch, algorithmic bytes per launch) of one V-cycle kernel."""
        ms, by = C.c_double(), C.c_double()
        _check(lib().fsigpu_gmg_time_kernel(self.h, self.KERNELS[which], level, reps, 1 if cold else 0,
                                            C.byref(ms), C.byref(by)))
        return ms.value, by.value

    def set_launch(self, level: int, which: str, lpr: int, unroll: int = 4):
        w = {"A": 0, "FS": 1, "AP": 2, "P": 3, "R": 4}[which]
        _check(lib().fsigpu_gmg_set_launch(self.h, level, w, lpr, unroll))

    def stream(self) -> int:
        """cudaStream_t (as int) all kernels of this hierarchy run on."""
        return lib().fsigpu_gmg_stream(self.h) or 0

    def apply(self, r) -> np.ndarray:
        r = _f64(r)
        z = np.empty(self.n)
        _check(lib().fsigpu_gmg_apply(self.h, r.ctypes.data, z.ctypes.data))
        return z

    def apply_dev(self, d_r: int, d_z: int):
        _check(lib().fsigpu_gmg_apply_dev(self.h, C.c_void_p(d_r), C.c_void_p(d_z), None))

    def fs_apply(self, level: int, r) -> np.ndarray:
        r = _f64(r)
        z = np.empty(self.levels[level].n)
        _check(lib().fsigpu_fs_apply(self.h, level, r.ctypes.data, z.ctypes.data))
        return z

    def coarse_solve(self, b) -> np.ndarray:
        b = _f64(b)
        x = np.empty(self.levels[0].n)
        _check(lib().fsigpu_coarse_solve(self.h, b.ctypes.data, x.ctypes.data))
        return x

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.fsigpu_gmg_destroy(self.h)
            self.h = None


@dataclass
class KrylovConfig:
    """krylov.hpp:42-47 (same defaults)."""
    restart: int = 60
    max_iters: int = 500
    rel_tol: float = 1e-8
    abs_tol: float = 1e-12


@dataclass
class GmresResult:
    """krylov.hpp:49-55 plus the V-cycle count and the true final residual."""
    x: np.ndarray
    history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    iterations: int = 0
    converged: bool = False
    breakdown: bool = False
    m_applies: int = 0
    true_residual: float = 0.0


class GmresSolver:
    """Device-resident FGMRES on diag(frame_scale) A_top, M = GMG(r / frame_scale)."""

    def __init__(self, gmg: GmgPreconditioner, frame_scale, restart: int = 30, graphs: bool = True):
        if restart < 1 or restart > 128:
            raise ValueError("gmres: restart must be in [1, 128]")
        self.gmg = gmg
        self.restart = restart
        self._scale = _f64(frame_scale)
        h = C.c_void_p()
        _check(lib().fsigpu_gmres_create(gmg.h, self._scale.ctypes.data, restart, C.byref(h)))
        self.h = h
        self.set_graphs(graphs)

    def set_graphs(self, on: bool):
        _check(lib().fsigpu_gmres_set_graphs(self.h, 1 if on else 0))

    def solve(self, b, cfg: KrylovConfig, x0=None) -> GmresResult:
        n = self.gmg.n
        b = _f64(b)
        if b.shape != (n,):
            raise ValueError("gmres: rhs size mismatch")
        if cfg.restart != self.restart:
            raise ValueError("gmres: solver built for a different restart")
        x = np.empty(n)
        hist = np.empty(cfg.max_iters + 2)
        res = GmresResultC()
        x0p = None if x0 is None else _f64(x0)
        _check(lib().fsigpu_gmres_solve(self.h, b.ctypes.data, None if x0p is None else x0p.ctypes.data,
                                        x.ctypes.data, cfg.max_iters, cfg.rel_tol, cfg.abs_tol,
                                        hist.ctypes.data, C.byref(res)))
        return GmresResult(x=x, history=hist[:res.n_history].copy(), iterations=res.iterations,
                           converged=bool(res.converged), breakdown=bool(res.breakdown),
                           m_applies=res.m_applies, true_residual=res.true_residual)

    def solve_dev(self, d_b: int, d_x: int, cfg: KrylovConfig) -> GmresResult:
        res = GmresResultC()
        _check(lib().fsigpu_gmres_solve_dev(self.h, C.c_void_p(d_b), C.c_void_p(d_x), cfg.max_iters,
                                            cfg.rel_tol, cfg.abs_tol, None, C.byref(res)))
        return GmresResult(x=np.zeros(0), iterations=res.iterations, converged=bool(res.converged),
                           breakdown=bool(res.breakdown), m_applies=res.m_applies,
                           true_residual=res.true_residual)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.fsigpu_gmres_destroy(self.h)
            self.h = None


def build_block_sets(level: Level, epb_as1: int = 0, epb_as2: int = 0, overlap: int = -1,
                     vanka: bool = False):
    """The level's Schwarz block sets built on the device from its mesh-side
    index maps (fsigpu_fs_sets_build / fsigpu_vanka_sets_build): returns a copy
    of the level with as1/as2, lumped and labels replaced (FsPreconditioner's
    sets, precond.cpp:119-269, or the Vanka sets, ordering.cpp:77-115)."""
    import copy
    init()
    m = level.mesh
    if m is None:
        raise ValueError("level has no mesh maps")
    epb1 = epb_as1 or int(m["epb_as1"][0])
    epb2 = epb_as2 or int(m["epb_as2"][0])
    ov = overlap if overlap >= 0 else int(m["overlap"][0])
    md = mesh_desc(m)
    h = C.c_void_p()
    if vanka:
        _check(lib().fsigpu_vanka_sets_build(level.n, C.byref(md), epb1, C.byref(h)))
    else:
        desc = level_descs([level, level])  # entry 1: a smoothed level (g1, n_us filled)
        _check(lib().fsigpu_fs_sets_build(C.byref(desc[1]), C.byref(md), epb1, epb2, ov, C.byref(h)))
    try:
        n1, l1, n2, l2, nus = (C.c_int() for _ in range(5))
        _check(lib().fsigpu_sets_counts(h, C.byref(n1), C.byref(l1), C.byref(n2), C.byref(l2), C.byref(nus)))
        p1, i1 = np.zeros(n1.value + 1, np.int32), np.zeros(max(l1.value, 1), np.int32)
        p2, i2 = np.zeros(n2.value + 1, np.int32), np.zeros(max(l2.value, 1), np.int32)
        lm = np.zeros(max(nus.value, 1))
        _check(lib().fsigpu_sets_copy(h, p1.ctypes.data, i1.ctypes.data, p2.ctypes.data, i2.ctypes.data,
                                      lm.ctypes.data))
        labels = [lib().fsigpu_sets_label(h, b).decode() for b in range(n1.value + n2.value)]
    finally:
        lib().fsigpu_sets_destroy(h)
    out = copy.copy(level)
    out.as1 = BlockSets(p1, i1[:l1.value].copy())
    out.as2 = BlockSets(p2, i2[:l2.value].copy())
    if not vanka:
        out.lumped = lm[:nus.value].copy()
    out.labels = labels
    return out


MODE_LU, MODE_INVERSE, MODE_ASSEMBLED = 0, 1, 2


def set_block_mode(mode: int):
    """Block-solve mode for GMG hierarchies created afterwards (fsigpu_set_block_mode)."""
    init()
    _check(lib().fsigpu_set_block_mode(mode))


def set_pdl(on: bool):
    """Programmatic dependent launch of the solve-path kernels (default off)."""
    init()
    _check(lib().fsigpu_set_pdl(1 if on else 0))


def launch_count() -> int:
    return int(lib().fsigpu_launch_count())


def gmres(gmg: GmgPreconditioner, frame_scale, b, cfg: KrylovConfig, x0=None) -> GmresResult:
    """gmres(a, m, b, cfg, x0) of krylov.hpp:61-62 for the driver's operators."""
    return GmresSolver(gmg, frame_scale, cfg.restart).solve(b, cfg, x0)


class Profile:
    """Accumulated per-kernel-class device time (CUDA events on the library stream)."""

    @staticmethod
    def enable(on: bool = True):
        _check(lib().fsigpu_profile_enable(1 if on else 0))

    @staticmethod
    def reset():
        _check(lib().fsigpu_profile_reset())

    @staticmethod
    def read():
        ms = np.zeros(6)
        n = np.zeros(6, np.int64)
        by = np.zeros(6)
        _check(lib().fsigpu_profile_read(ms.ctypes.data, n.ctypes.data, by.ctypes.data))
        return {k: dict(ms=float(ms[i]), launches=int(n[i]), bytes=float(by[i]))
                for i, k in enumerate(KERNEL_CLASSES)}

    @staticmethod
    def read_level(cls: str, level: int):
        """Sums of one kernel class on one GMG level (in-solve per-launch events)."""
        ms, by = C.c_double(), C.c_double()
        n = C.c_longlong()
        _check(lib().fsigpu_profile_read_level(KERNEL_CLASSES.index(cls), level, C.byref(ms), C.byref(n),
                                               C.byref(by)))
        return dict(ms=ms.value, launches=n.value, bytes=by.value)


class Stamps:
    """Device-clock launch stamps: kernel durations INSIDE the captured
    restart-cycle graph (last CTA exit minus dependency release), where CUDA
    events cannot bracket a launch. enable() resets the counters and makes the
    solvers re-capture their graphs."""

    @staticmethod
    def enable(on: bool = True):
        _check(lib().fsigpu_stamps_enable(1 if on else 0))

    @staticmethod
    def read(cls: str, level: int, sub: int = 0):
        us = C.c_double()
        n = C.c_longlong()
        _check(lib().fsigpu_stamps_read(KERNEL_CLASSES.index(cls), level, sub, C.byref(us), C.byref(n)))
        return dict(us=us.value, launches=n.value)
