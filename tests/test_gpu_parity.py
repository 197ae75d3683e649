"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and
the reference's golden outputs on identical inputs."""
import numpy as np
import pytest

import oracle as O
from paper_1909_13201_b200 import fsigpu

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def split_blocks(gb):
    sizes = gb["sizes"]
    mats, rhs, xs = [], [], []
    o = r = 0
    for m in sizes:
        m = int(m)
        mats.append(gb["a"][o:o + m * m].reshape(m, m))
        rhs.append(gb["b"][r:r + m])
        xs.append(gb["x"][r:r + m])
        o += m * m
        r += m
    return sizes, mats, rhs, xs


# ---------------------------------------------------------------- SpMV
def test_spmv_known_answers():
    # tests/unit_linalg.cpp:156-164
    from paper_1909_13201_b200.problem import Csr
    a = Csr(2, 2, np.array([0, 2, 4], np.int32), np.array([0, 1, 0, 1], np.int32), np.array([4., 1., 1., 3.]))
    assert np.array_equal(fsigpu.SparseMatrix(a).multiply([1, 2]), [6, 7])
    eye = Csr(3, 3, np.arange(4, dtype=np.int32), np.arange(3, dtype=np.int32), np.ones(3))
    assert np.array_equal(fsigpu.SparseMatrix(eye).multiply([1, 2, 3]), [1, 2, 3])
    zero = Csr(4, 4, np.zeros(5, np.int32), np.zeros(0, np.int32), np.zeros(0))
    assert np.array_equal(fsigpu.SparseMatrix(zero).multiply([1, -2, 3, -4]), [0, 0, 0, 0])
    with pytest.raises(ValueError):
        fsigpu.SparseMatrix(a).multiply([1, 2, 3])


def test_spmv_level_matrices(cfg0):
    for lv in cfg0.levels:
        for M in [lv.A] + ([lv.P, lv.R] if lv.P is not None else []):
            x = np.random.default_rng(3).uniform(-1, 1, M.cols)
            y = fsigpu.SparseMatrix(M).multiply(x)
            yo = O.spmv(M, x)
            assert np.max(np.abs(y - yo)) <= 1e-13 * max(1.0, np.max(np.abs(yo)))
    g = cfg0.golden
    y = fsigpu.SparseMatrix(cfg0.levels[-1].A).multiply(g["golden/spmv_x"])
    assert rel(y, g["golden/spmv_y"]) < 1e-14


# ---------------------------------------------------------------- dense LU
def test_dense_lu_known_answers():
    # tests/unit_linalg.cpp:229-247
    B = fsigpu.DenseBlocks.from_dense([np.eye(2), np.array([[4., 1.], [1., 3.]])])
    x = B.solve(np.array([5., 6., 1., 2.]))
    assert np.array_equal(x[:2], [5, 6])
    assert abs(x[2] - 1 / 11) <= 1e-14 / 11 and abs(x[3] - 7 / 11) <= 1e-14 * 7 / 11
    with pytest.raises(fsigpu.SingularBlockError, match="singular block: wall-block"):
        fsigpu.DenseBlocks.from_dense([np.eye(3), np.ones((2, 2))], labels=["ok", "wall-block"])


def test_dense_lu_golden_blocks_bitexact(golden_blocks):
    sizes, mats, rhs, xs = split_blocks(golden_blocks)
    B = fsigpu.DenseBlocks.from_dense(mats)
    lus = B.lu(sizes)
    for m, (lu, piv) in zip(mats, lus):
        lo, po = O.dense_factor(m)
        assert np.array_equal(piv, po), "pivot sequence differs from DenseFactorization"
        assert np.array_equal(lu, lo), "LU factors not bit-identical to DenseFactorization"
    x = B.solve(np.concatenate(rhs))
    o = 0
    for m, xr in zip(sizes, xs):
        assert rel(x[o:o + m], xr) <= 1e-12
        o += m


def test_fs_blocks_vs_reference(cfg0):
    """Per-block AS solves of the real config-0 fine-level FS blocks within
    1e-12 relative of DenseFactorization::solve (golden from the reference)."""
    top = cfg0.levels[-1]
    A = fsigpu.SparseMatrix(top.A)
    sets = [top.as1.idx[top.as1.ptr[b]:top.as1.ptr[b + 1]] for b in range(top.as1.n)]
    sets += [top.as2.idx[top.as2.ptr[b]:top.as2.ptr[b + 1]] + top.g1 for b in range(top.as2.n)]
    B = fsigpu.DenseBlocks.from_csr(A, sets)
    rhs, xs = cfg0.golden["golden/block_rhs"], cfg0.golden["golden/block_x"]
    x = B.solve(rhs)
    o = 0
    worst = 0.0
    for s in sets:
        m = len(s)
        worst = max(worst, rel(x[o:o + m], xs[o:o + m]))
        o += m
    assert worst <= 1e-12, worst
    # factors bit-identical to the oracle's DenseFactorization
    lus = B.lu([len(s) for s in sets])
    for k in [0, 17, len(sets) // 2, len(sets) - 1]:
        lo, po = O.dense_factor(O.extract_block(top.A, sets[k]))
        assert np.array_equal(lus[k][0], lo) and np.array_equal(lus[k][1], po)


# ---------------------------------------------------------------- FS / GMG
MODES = pytest.mark.parametrize("mode", [fsigpu.MODE_LU, fsigpu.MODE_INVERSE], ids=["lu", "inverse"])


def gmg(levels, mode):
    fsigpu.set_block_mode(mode)
    try:
        return fsigpu.GmgPreconditioner(levels)
    finally:
        fsigpu.set_block_mode(fsigpu.MODE_INVERSE)


@MODES
def test_fs_apply_vs_reference(cfg0, mode):
    G = gmg(cfg0.levels, mode)
    g = cfg0.golden
    z = G.fs_apply(len(cfg0.levels) - 1, g["golden/fs_r"])
    assert rel(z, g["golden/fs_z_add"]) <= 1e-12


def test_coarse_solve(cfg0):
    G = fsigpu.GmgPreconditioner(cfg0.levels)
    g = cfg0.golden
    assert rel(G.coarse_solve(g["golden/coarse_b"]), g["golden/coarse_x"]) <= 1e-9


@MODES
def test_vcycle_vs_reference(cfg0, mode):
    G = gmg(cfg0.levels, mode)
    g = cfg0.golden
    z = G.apply(g["golden/vcycle_r"])
    assert rel(z, g["golden/vcycle_z_add"]) <= 1e-9
    OG = O.OracleGmg(cfg0.levels)
    assert rel(z, OG.apply(g["golden/vcycle_r"])) <= 1e-9


@MODES
def test_gmres_cfg0_parity(cfg0, mode):
    """North-star parity: iterations within +-1 and final relative residual
    within 1e-8 of the additive oracle's on identical inputs."""
    G = gmg(cfg0.levels, mode)
    cfg = fsigpu.KrylovConfig(restart=30, max_iters=2000, rel_tol=1e-10, abs_tol=1e-300)
    res = fsigpu.gmres(G, cfg0.frame_scale, cfg0.b, cfg)
    g = cfg0.golden
    ref_its = int(g["gmres_add/iterations"][0])
    assert res.converged
    assert abs(res.iterations - ref_its) <= 1, (res.iterations, ref_its)
    r0 = res.history[0]
    ref_rel = g["gmres_add/true_residual"][0] / g["gmres_add/history"][0]
    assert abs(res.true_residual / r0 - ref_rel) <= 1e-8
    assert rel(res.x, g["gmres_add/x"]) <= 1e-6
