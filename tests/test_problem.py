"""CPU tier: solve-phase inputs (FSIX fixtures) are well formed and carry
the reference driver's invariants (driver.cpp:206-272, precond.cpp:119-269)."""
import numpy as np

from paper_1909_13201_b200 import fsix
from paper_1909_13201_b200.problem import level_descs


def check_csr(a):
    assert a.ptr[0] == 0 and np.all(np.diff(a.ptr) >= 0)
    for i in range(a.rows):
        c = a.idx[a.ptr[i]:a.ptr[i + 1]]
        assert np.all(np.diff(c) > 0) and (len(c) == 0 or (c[0] >= 0 and c[-1] < a.cols))
    assert np.all(np.isfinite(a.val))


def test_fsix_roundtrip(tmp_path):
    arrs = {"a": np.arange(5, dtype=np.float64), "b": np.array([1, -2], np.int32),
            "c": np.array([0, 1, 1], np.uint8)}
    p = tmp_path / "t.fsix"
    fsix.save(str(p), arrs)
    back = fsix.load(str(p))
    for k, v in arrs.items():
        assert np.array_equal(back[k], v) and back[k].dtype == v.dtype


def test_chan_fixture_invariants(chan):
    L = chan.levels
    assert len(L) == 2
    for l, lv in enumerate(L):
        check_csr(lv.A)
        assert lv.A.rows == lv.A.cols == lv.n
        if l == 0:
            continue
        check_csr(lv.P)
        check_csr(lv.R)
        assert lv.P.rows == lv.n and lv.P.cols == L[l - 1].n
        assert lv.R.rows == L[l - 1].n and lv.R.cols == lv.n
        # FS group sizes and the lumped solid-velocity mass (precond.cpp:231-245)
        assert 0 < lv.g1 < lv.n and 0 <= lv.n_us <= lv.n - lv.g1
        assert np.all(lv.lumped > 0)
        for bs, lo, hi in [(lv.as1, 0, lv.g1), (lv.as2, lv.n_us, lv.n - lv.g1)]:
            for b in range(bs.n):
                s = bs.idx[bs.ptr[b]:bs.ptr[b + 1]]
                assert len(s) > 0 and np.all(np.diff(s) > 0) and s[0] >= lo and s[-1] < hi
        # blocks never contain constrained positions (precond.cpp:90-97)
        frame = np.concatenate([lv.as1.idx, lv.as2.idx + lv.g1])
        assert not np.any(lv.row_mask[frame] & lv.col_mask[frame])
    # RHS zero on constrained rows, positive row scales (D9)
    assert np.all(chan.b[L[-1].row_mask == 1] == 0.0)
    assert np.all(chan.frame_scale > 0)


def test_level_descs_layout(chan):
    d = level_descs(chan.levels)
    assert d[0].n == chan.levels[0].n and d[1].nc == chan.levels[0].n
    assert d[1].as1_n == chan.levels[1].as1.n and d[1].g1 == chan.levels[1].g1
