"""Solve-phase inputs of one linear system (one first-Newton Jacobian).

Mirrors what the reference driver hands to the solve layer
(proj/src/driver.cpp:206-272): per level the J2-frame Jacobian
(``GmgLevel::a``), the constraint masks (``constrained_rows/cols``,
driver.cpp:250-255), the transfers P/R (``TransferPair``, gmg.cpp:77-136),
and for levels >= 1 the FS smoother data: group sizes, the lumped
solid-velocity mass (precond.cpp:231-245) and the AS1 / AS2 block index sets
(precond.cpp:163-268).  On the finest level the outer system is the
row-equilibrated frame operator (driver.cpp:150-186,259-262) with RHS ``b``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from . import fsix


@dataclass
class Csr:
    rows: int
    cols: int
    ptr: np.ndarray
    idx: np.ndarray
    val: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.ptr[-1])

    @staticmethod
    def from_arch(a: Dict[str, np.ndarray], pre: str) -> "Csr":
        return Csr(int(a[pre + "/rows"][0]), int(a[pre + "/cols"][0]),
                   np.ascontiguousarray(a[pre + "/ptr"], np.int32),
                   np.ascontiguousarray(a[pre + "/idx"], np.int32),
                   np.ascontiguousarray(a[pre + "/val"], np.float64))

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.val, self.idx, self.ptr), shape=(self.rows, self.cols))


@dataclass
class BlockSets:
    ptr: np.ndarray
    idx: np.ndarray

    @property
    def n(self) -> int:
        return len(self.ptr) - 1

    def sizes(self) -> np.ndarray:
        return np.diff(self.ptr)


@dataclass
class Level:
    n: int
    A: Csr
    row_mask: np.ndarray
    col_mask: np.ndarray
    P: Optional[Csr] = None
    R: Optional[Csr] = None
    g1: int = 0
    n_us: int = 0
    lumped: Optional[np.ndarray] = None
    as1: Optional[BlockSets] = None
    as2: Optional[BlockSets] = None
    labels: Optional[List[str]] = None  # reference IndexSet labels, AS1 then AS2 blocks
    # mesh-side index maps of the block construction (fsigpu_mesh_desc), if exported
    mesh: Optional[Dict[str, np.ndarray]] = None


@dataclass
class Problem:
    name: str
    levels: List[Level]
    frame_scale: np.ndarray
    b: np.ndarray
    golden: Dict[str, np.ndarray] = field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.levels[-1].n


def load_case(path: str, name: str = "") -> Problem:
    a = fsix.load(path)
    L = int(a["levels"][0])
    levels = []
    for l in range(L):
        p = f"L{l}"
        A = Csr.from_arch(a, p + "/A")
        lv = Level(n=A.rows, A=A, row_mask=a[p + "/row_mask"].astype(np.uint8),
                   col_mask=a[p + "/col_mask"].astype(np.uint8))
        if l > 0:
            lv.P = Csr.from_arch(a, p + "/P")
            lv.R = Csr.from_arch(a, p + "/R")
            lv.g1 = int(a[p + "/g1"][0])
            lv.n_us = int(a[p + "/n_us"][0])
            lv.lumped = a[p + "/lumped"].astype(np.float64)
            lv.as1 = BlockSets(a[p + "/as1/ptr"].astype(np.int32), a[p + "/as1/idx"].astype(np.int32))
            lv.as2 = BlockSets(a[p + "/as2/ptr"].astype(np.int32), a[p + "/as2/idx"].astype(np.int32))
            if p + "/as1/labels" in a:
                lv.labels = [t for k in ("as1", "as2")
                             for t in bytes(a[f"{p}/{k}/labels"]).decode().split("\n")[:-1]]
        if p + "/mesh/element_nodes" in a:
            lv.mesh = {k[len(p) + 6:]: v for k, v in a.items() if k.startswith(p + "/mesh/")}
        levels.append(lv)
    golden = {k: v for k, v in a.items() if k.startswith(("golden/", "gmres_", "gmres/", "setup/"))}
    return Problem(name=name or path, levels=levels, frame_scale=a["frame_scale"].astype(np.float64),
                   b=a["b"].astype(np.float64), golden=golden)


class LevelDesc(C.Structure):
    """C layout shared by ``fsigpu_level_desc`` (include/fsigpu.h) and the
    oracle's ``orc_level_desc`` (oracle/fsi_oracle.h)."""
    _fields_ = [
        ("n", C.c_int),
        ("a_ptr", C.c_void_p), ("a_idx", C.c_void_p), ("a_val", C.c_void_p),
        ("row_mask", C.c_void_p), ("col_mask", C.c_void_p),
        ("nc", C.c_int),
        ("p_ptr", C.c_void_p), ("p_idx", C.c_void_p), ("p_val", C.c_void_p),
        ("r_ptr", C.c_void_p), ("r_idx", C.c_void_p), ("r_val", C.c_void_p),
        ("g1", C.c_int), ("n_us", C.c_int),
        ("lumped", C.c_void_p),
        ("as1_n", C.c_int), ("as1_ptr", C.c_void_p), ("as1_idx", C.c_void_p),
        ("as2_n", C.c_int), ("as2_ptr", C.c_void_p), ("as2_idx", C.c_void_p),
    ]


class MeshDesc(C.Structure):
    """C layout of ``fsigpu_mesh_desc`` (include/fsigpu.h)."""
    _fields_ = [
        ("n_elements", C.c_int), ("n_nodes", C.c_int), ("nodes_per_element", C.c_int),
        ("dim", C.c_int), ("p_per_element", C.c_int),
        ("element_nodes", C.c_void_p), ("elem_solid", C.c_void_p), ("node_solid", C.c_void_p),
        ("d_pos", C.c_void_p), ("u_pos", C.c_void_p), ("p_pos", C.c_void_p), ("drop", C.c_void_p),
    ]


def mesh_desc(m: Dict[str, np.ndarray], npe: int = 9, dim: int = 2, ppe: int = 3) -> MeshDesc:
    """MeshDesc over the (kept-alive) arrays of an exported level mesh (2D Q2
    by default; 3D archives carry nodes_per_element / dim / p_per_element)."""
    npe = int(m["nodes_per_element"][0]) if "nodes_per_element" in m else npe
    dim = int(m["dim"][0]) if "dim" in m else dim
    ppe = int(m["p_per_element"][0]) if "p_per_element" in m else ppe
    d = MeshDesc()
    d.n_elements = len(m["elem_solid"])
    d.n_nodes = len(m["node_solid"])
    d.nodes_per_element, d.dim, d.p_per_element = npe, dim, ppe
    d.element_nodes, d.elem_solid, d.node_solid = (m["element_nodes"].ctypes.data, m["elem_solid"].ctypes.data,
                                                   m["node_solid"].ctypes.data)
    d.d_pos, d.u_pos, d.p_pos = m["d_pos"].ctypes.data, m["u_pos"].ctypes.data, m["p_pos"].ctypes.data
    d.drop = m["drop"].ctypes.data if "drop" in m else None
    return d


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def level_descs(levels: List[Level]):
    """Array of LevelDesc pointing into the (kept-alive) numpy buffers."""
    arr = (LevelDesc * len(levels))()
    for l, lv in enumerate(levels):
        d = arr[l]
        d.n = lv.n
        d.a_ptr, d.a_idx, d.a_val = _p(lv.A.ptr), _p(lv.A.idx), _p(lv.A.val)
        d.row_mask, d.col_mask = _p(lv.row_mask), _p(lv.col_mask)
        if l > 0:
            d.nc = lv.P.cols
            d.p_ptr, d.p_idx, d.p_val = _p(lv.P.ptr), _p(lv.P.idx), _p(lv.P.val)
            d.r_ptr, d.r_idx, d.r_val = _p(lv.R.ptr), _p(lv.R.idx), _p(lv.R.val)
            d.g1, d.n_us = lv.g1, lv.n_us
            d.lumped = _p(lv.lumped)
            d.as1_n, d.as1_ptr, d.as1_idx = lv.as1.n, _p(lv.as1.ptr), _p(lv.as1.idx)
            d.as2_n, d.as2_ptr, d.as2_idx = lv.as2.n, _p(lv.as2.ptr), _p(lv.as2.idx)
    return arr
