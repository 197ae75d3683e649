"""Pin the C restatement oracle (oracle/fsi_oracle.c) against the reference:
known-answer tests restated from the reference's own unit tests and golden
outputs of the unmodified reference library (tests/golden/*.fsix, written by
oracle/ref_harness/harness.cpp — regenerate with oracle/make_golden.sh)."""
import numpy as np
import pytest

import oracle as O
from paper_1909_13201_b200.problem import Csr


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def csr_from_dense(d):
    d = np.asarray(d, float)
    ptr, idx, val = [0], [], []
    for i in range(d.shape[0]):
        for j in range(d.shape[1]):
            if d[i, j] != 0.0:
                idx.append(j)
                val.append(d[i, j])
        ptr.append(len(idx))
    return Csr(d.shape[0], d.shape[1], np.array(ptr, np.int32), np.array(idx, np.int32), np.array(val))


# ---- tests/unit_linalg.cpp:156-187 (SpMV)
def test_spmv_known_answers():
    a = csr_from_dense([[4, 1], [1, 3]])
    assert np.array_equal(O.spmv(a, [1, 2]), [6, 7])
    assert np.array_equal(O.spmv(csr_from_dense(np.eye(3)), [1, 2, 3]), [1, 2, 3])
    z = Csr(4, 4, np.zeros(5, np.int32), np.zeros(0, np.int32), np.zeros(0))
    assert np.array_equal(O.spmv(z, [1, -2, 3, -4]), [0, 0, 0, 0])


def test_spmv_linearity():
    rng = np.random.default_rng(20240901)
    for _ in range(5):
        n = 17
        d = np.zeros((n, n))
        for i in range(n):
            for _k in range(5):
                d[i, rng.integers(0, n)] += rng.uniform(-1, 1)
        a = csr_from_dense(d)
        x, y = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        al, be = 0.37, -1.21
        lhs = O.spmv(a, al * x + be * y)
        rhs = al * O.spmv(a, x) + be * O.spmv(a, y)
        assert np.all(np.abs(lhs - rhs) <= 1e-13 * np.maximum(1.0, np.abs(rhs)))


# ---- tests/unit_linalg.cpp:229-261 (dense LU)
def test_dense_lu_known_answers():
    lu, piv = O.dense_factor(np.eye(2))
    assert np.array_equal(O.dense_solve(lu, piv, [5, 6]), [5, 6])
    lu, piv = O.dense_factor(np.array([[4., 1.], [1., 3.]]))
    x = O.dense_solve(lu, piv, [1, 2])
    assert x[0] == pytest.approx(1 / 11, rel=1e-14) and x[1] == pytest.approx(7 / 11, rel=1e-14)
    with pytest.raises(ZeroDivisionError):
        O.dense_factor(np.ones((2, 2)))
    rng = np.random.default_rng(1)
    n = 40
    r = rng.uniform(-1, 1, (n, n)) + n * np.eye(n)
    b = rng.uniform(-1, 1, n)
    lu, piv = O.dense_factor(r)
    assert rel(r @ O.dense_solve(lu, piv, b), b) <= 1e-10


def test_dense_lu_golden_bitexact(golden_blocks):
    """DenseFactorization::solve golden outputs (dominant, pivoting, graded
    blocks up to m = 162) reproduced bit for bit by the restatement."""
    g = golden_blocks
    o = r = 0
    for m, kind in zip(g["sizes"], g["kinds"]):
        m = int(m)
        a = g["a"][o:o + m * m].reshape(m, m)
        lu, piv = O.dense_factor(a)
        x = O.dense_solve(lu, piv, g["b"][r:r + m])
        assert np.array_equal(x, g["x"][r:r + m]), (m, kind)
        o += m * m
        r += m
    assert int(g["singular_thrown"][0]) == 1
    assert bytes(g["singular_msg"]).decode() == "singular block: wall-block"


def test_pivoting_exercised(golden_blocks):
    g = golden_blocks
    o = 0
    swaps = 0
    for m in g["sizes"]:
        m = int(m)
        _, piv = O.dense_factor(g["a"][o:o + m * m].reshape(m, m))
        swaps += int(np.sum(piv != np.arange(m)))
        o += m * m
    assert swaps > 0


# ---- FS / GMG / GMRES against the reference (channel fixture of the
# reference's own tests, tests/unit_solver.cpp:48-60, first Newton Jacobian)
def test_fs_apply_bitexact_chan(chan):
    G = O.OracleGmg(chan.levels)
    g = chan.golden
    z = G.fs_apply(len(chan.levels) - 1, g["golden/fs_r"])
    assert np.array_equal(z, g["golden/fs_z_add"])


def test_block_solves_bitexact_chan(chan):
    top = chan.levels[-1]
    sets = [top.as1.idx[top.as1.ptr[b]:top.as1.ptr[b + 1]] for b in range(top.as1.n)]
    sets += [top.as2.idx[top.as2.ptr[b]:top.as2.ptr[b + 1]] + top.g1 for b in range(top.as2.n)]
    rhs, xs = chan.golden["golden/block_rhs"], chan.golden["golden/block_x"]
    o = 0
    for s in sets:
        m = len(s)
        lu, piv = O.dense_factor(O.extract_block(top.A, s))
        assert np.array_equal(O.dense_solve(lu, piv, rhs[o:o + m]), xs[o:o + m])
        o += m


def test_spmv_coarse_vcycle_chan(chan):
    g = chan.golden
    top = chan.levels[-1]
    assert np.array_equal(O.spmv(top.A, g["golden/spmv_x"]), g["golden/spmv_y"])
    G = O.OracleGmg(chan.levels)
    assert rel(G.coarse_solve(g["golden/coarse_b"]), g["golden/coarse_x"]) <= 1e-10
    assert rel(G.apply(g["golden/vcycle_r"]), g["golden/vcycle_z_add"]) <= 1e-10


def test_gmres_chan_matches_reference(chan):
    g = chan.golden
    G = O.OracleGmg(chan.levels)
    rtol = float(g["gmres/rel_tol"][0]) if "gmres/rel_tol" in g else 1e-8
    r = G.gmres(chan.frame_scale, chan.b, restart=30, max_iters=300, rel_tol=rtol)
    assert r["iterations"] == int(g["gmres_add/iterations"][0])
    assert r["m_applies"] == int(g["gmres_add/m_applies"][0])
    # The restated coarse solve (dense LU) differs from SparseLu by rounding.
    # This SI-unit channel system is badly conditioned, so the late
    # recurrence residuals of the restarted GMRES drift (up to O(1) relative
    # near the stagnation plateau) while the iterate itself agrees to 1e-11.
    h, hr = r["history"], g["gmres_add/history"]
    assert len(h) == len(hr)
    assert np.all(np.abs(h[:10] - hr[:10]) <= 1e-6 * hr[:10])
    assert rel(r["x"], g["gmres_add/x"]) <= 1e-9


def test_gmres_identity_and_exact_preconditioner():
    """tests/unit_linalg.cpp:331-397 analogue on a 1-level hierarchy: the
    coarse direct solve as M makes GMRES converge in one iteration."""
    from paper_1909_13201_b200.problem import Level
    a = csr_from_dense([[4, 1, 0], [1, 3, 1], [0, 1, 2]])
    lv = Level(n=3, A=a, row_mask=np.zeros(3, np.uint8), col_mask=np.zeros(3, np.uint8))
    G = O.OracleGmg([lv])
    r = G.gmres(np.ones(3), np.array([1.0, 2.0, 3.0]), restart=30, max_iters=10, rel_tol=1e-12)
    assert r["converged"] and r["iterations"] == 1
    assert rel(O.spmv(a, r["x"]), [1, 2, 3]) <= 1e-12


@pytest.mark.slow
def test_oracle_cfg0_matches_reference(cfg0):
    g = cfg0.golden
    G = O.OracleGmg(cfg0.levels)
    z = G.fs_apply(len(cfg0.levels) - 1, g["golden/fs_r"])
    assert np.array_equal(z, g["golden/fs_z_add"])
    r = G.gmres(cfg0.frame_scale, cfg0.b, restart=30, max_iters=2000, rel_tol=1e-10, abs_tol=1e-300)
    assert r["iterations"] == int(g["gmres_add/iterations"][0])


# ---- the shipped multiplicative FS / AS smoothers (precond.cpp:59-77,
# 99-117, 271-303) and their multicolour reordering (the GPU's)
@pytest.mark.parametrize("case", ["chan", "chan_as"])
def test_multiplicative_sweep_bitexact(case, request):
    """The restated multiplicative sweep in the reference's block order is
    bit-identical to FsPreconditioner::apply / AsPreconditioner::apply."""
    P = request.getfixturevalue(case)
    g = P.golden
    G = O.OracleGmg(P.levels, fs="multiplicative")
    assert np.array_equal(G.fs_apply(len(P.levels) - 1, g["golden/fs_r"]), g["golden/fs_z_mult"])


@pytest.mark.parametrize("case", ["cfg0", "cfg0_as"])
def test_multiplicative_gmres_matches_reference(case, request):
    """GMRES(30) with the restated shipped multiplicative smoother on config 0
    (FS: the reference's 76 iterations; AS: 72) matches the reference's solve.
    (On the SI-unit channel case the recurrence residuals drift at 1e-7 from
    step 7 on, from the coarse solve's rounding, and the iteration count near
    the 1e-8 floor moves by a few.)"""
    P = request.getfixturevalue(case)
    g = P.golden
    G = O.OracleGmg(P.levels, fs="multiplicative")
    assert np.array_equal(G.fs_apply(len(P.levels) - 1, g["golden/fs_r"]), g["golden/fs_z_mult"])
    r = G.gmres(P.frame_scale, P.b, restart=30, max_iters=2000, rel_tol=1e-10, abs_tol=1e-300)
    assert r["converged"]
    assert abs(r["iterations"] - int(g["gmres_mult/iterations"][0])) <= 1, (r["iterations"],
                                                                           int(g["gmres_mult/iterations"][0]))
    assert rel(r["x"], g["gmres_mult/x"]) <= 1e-6


def test_multicolour_order_properties(chan):
    """The multicolour order is a valid multiplicative ordering: a linear
    map, different from the reference's block order only by the order of the
    blocks (same result on block-diagonal systems), converging like it."""
    top = len(chan.levels) - 1
    Gc = O.OracleGmg(chan.levels, fs="multicolour")
    Gm = O.OracleGmg(chan.levels, fs="multiplicative")
    assert 2 <= Gc.colours(top, 1) <= 16 and 2 <= Gc.colours(top, 2) <= 16
    rng = np.random.default_rng(3)
    u, v = rng.uniform(-1, 1, chan.n), rng.uniform(-1, 1, chan.n)
    zu, zv, zs = Gc.fs_apply(top, u), Gc.fs_apply(top, v), Gc.fs_apply(top, 2.0 * u - 3.0 * v)
    assert rel(zs, 2.0 * zu - 3.0 * zv) <= 1e-12
    assert not np.array_equal(zu, Gm.fs_apply(top, u))
    rc = Gc.gmres(chan.frame_scale, chan.b, restart=30, max_iters=300, rel_tol=1e-8)
    rm = Gm.gmres(chan.frame_scale, chan.b, restart=30, max_iters=300, rel_tol=1e-8)
    assert rc["converged"] and rm["converged"] and abs(rc["iterations"] - rm["iterations"]) <= 5


# ---- AS (Vanka, J1) smoother: additive sweep over the reference's
# AsPreconditioner blocks (precond.cpp:99-117; build_vanka_blocks,
# ordering.cpp:77-115) -- the "pure DD" smoother of BASELINE configs 0/4
def test_as_smoother_chan_matches_reference(chan_as):
    g = chan_as.golden
    top = chan_as.levels[-1]
    assert top.g1 == top.n and top.n_us == 0 and top.as2.n == 0
    G = O.OracleGmg(chan_as.levels)
    assert np.array_equal(G.fs_apply(1, g["golden/fs_r"]), g["golden/fs_z_add"])
    assert rel(G.apply(g["golden/vcycle_r"]), g["golden/vcycle_z_add"]) <= 1e-10
    r = G.gmres(chan_as.frame_scale, chan_as.b, restart=30, max_iters=300, rel_tol=1e-8)
    assert r["iterations"] == int(g["gmres_add/iterations"][0])
    assert rel(r["x"], g["gmres_add/x"]) <= 1e-9


# ---- FGMRES and the GMRES(1) smoother (BASELINE configs[0])
def test_fgmres_equals_gmres_for_linear_smoother(chan):
    """For the linear Richardson V-cycle the flexible variant is the same
    method: same iteration count, iterate to rounding."""
    G = O.OracleGmg(chan.levels)
    a = G.gmres(chan.frame_scale, chan.b, restart=30, max_iters=300, rel_tol=1e-8)
    f = G.gmres(chan.frame_scale, chan.b, restart=30, max_iters=300, rel_tol=1e-8, flexible=True)
    assert abs(a["iterations"] - f["iterations"]) <= 1
    assert f["converged"]
    # one M apply per Arnoldi step only (no restart-end M(Vy))
    assert f["m_applies"] == f["iterations"]
    assert rel(f["x"], a["x"]) <= 1e-8


def test_gmres1_smoother_properties(chan, cfg0):
    """GMRES(1) smoothing is homogeneous of degree 1 (alpha is scale
    invariant: exactly so for a power-of-two scale) but not additive, and
    FGMRES converges with it on config 0 (197 iterations; Richardson: 103).
    On the SI-unit channel it stagnates (relres ~0.5 after 300 its)."""
    G = O.OracleGmg(chan.levels, smoother="gmres1")
    r = chan.golden["golden/vcycle_r"]
    z = G.apply(r)
    assert np.array_equal(G.apply(4.0 * r), 4.0 * z)
    rng = np.random.default_rng(7)
    r2 = rng.uniform(-1, 1, len(r)) * (np.abs(r) > 0)
    assert rel(G.apply(r + r2), z + G.apply(r2)) > 1e-6
    # zero input -> zero output (alpha = 0 when w = 0)
    assert not np.any(G.apply(np.zeros_like(r)))
    G0 = O.OracleGmg(cfg0.levels, smoother="gmres1")
    f = G0.gmres(cfg0.frame_scale, cfg0.b, restart=30, max_iters=400, rel_tol=1e-10, flexible=True)
    assert f["converged"] and 150 <= f["iterations"] <= 250, f["iterations"]


def test_gmres1_step_minimises_level_residual(chan):
    """One GMRES(1) pre-smoothing step from x = 0 (pre=1, post=0 on a
    2-level hierarchy) never increases the level residual norm, and does no
    worse than the damped Richardson step."""
    lv = chan.levels
    top = lv[-1]
    r = chan.golden["golden/vcycle_r"]
    A = top.A.to_scipy()
    Gm = O.OracleGmg(lv, smoother="gmres1")
    Gr = O.OracleGmg(lv)
    z_fs = Gr.fs_apply(len(lv) - 1, r)
    w = A @ z_fs
    alpha = (w @ r) / (w @ w)
    # closed form of the minimal-residual step vs Richardson omega = 0.7
    res_mr = np.linalg.norm(r - alpha * w)
    res_rich = np.linalg.norm(r - 0.7 * w)
    assert res_mr <= np.linalg.norm(r)
    assert res_mr <= res_rich * (1 + 1e-12)
    del Gm
