"""I/O formats of the reference toolchain, host-only:
SLW1 raw fields (inc/field_io.hpp:12-76) against a fixture written by the
reference's own write_slw1, and the SolveReport CSV (inc/krylov.hpp:26-34).
UNW1 checkpoints are covered in test_paper_net.py."""
import io
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def hg():
    from paper_2203_11025_b200 import build, helmgpu
    build.build()
    return helmgpu


def test_slw1_matches_reference_file(hg, tmp_path):
    from oracle import oracle as O
    k2 = O.make_medium(24, 16, 99)  # the field the fixture was written from
    path = os.path.join(GOLD, "medium_24x16.slw")
    f = hg.read_slw1(path)
    assert f.shape == (16, 24)
    assert np.array_equal(f, k2.astype(np.float32).astype(np.float64))
    out = tmp_path / "w.slw"
    hg.write_slw1(out, k2)
    assert out.read_bytes() == open(path, "rb").read()


def test_slw1_errors(hg, tmp_path):
    bad = tmp_path / "bad.slw"
    bad.write_bytes(b"SLW2" + b"\0" * 12)
    with pytest.raises(RuntimeError, match="bad SLW1"):
        hg.read_slw1(bad)
    good = open(os.path.join(GOLD, "medium_24x16.slw"), "rb").read()
    trunc = tmp_path / "trunc.slw"
    trunc.write_bytes(good[:-4])
    with pytest.raises(RuntimeError, match="truncated"):
        hg.read_slw1(trunc)
    with pytest.raises(RuntimeError, match="cannot open"):
        hg.read_slw1(tmp_path / "missing.slw")


def test_slw1_roundtrip_through_reference(hg, tmp_path):
    from oracle import oracle as O
    if not O.have_ref():
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    import ctypes as C
    R = O.ref()
    f = np.random.default_rng(3).random((5, 7))
    hg.write_slw1(tmp_path / "a.slw", f)
    nx, ny = C.c_int(), C.c_int()
    g = np.zeros((5, 7))
    assert R.hr_read_slw1(str(tmp_path / "a.slw").encode(), C.byref(nx), C.byref(ny), O._p(g)) == 0
    assert (nx.value, ny.value) == (7, 5) and np.array_equal(g, f.astype(np.float32))


def test_solve_report_csv(hg):
    rep = hg.SolveReport([np.array([2.0, 1.0, 0.5]), np.array([3.0, 1.0, 3e-7])], [2, 2], [True, False],
                         [False, False])
    s = io.StringIO()
    rep.write_csv(s)
    lines = s.getvalue().splitlines()
    assert lines[0] == "iter,rhs_index,relative_residual"
    # std::ostream default formatting (6 significant digits), inc/krylov.hpp:26-34
    assert lines[1:] == ["0,0,1", "1,0,0.5", "2,0,0.25", "0,1,1", "1,1,0.333333", "2,1,1e-07"]
