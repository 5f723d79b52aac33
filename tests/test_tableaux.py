"""Host tableau algebra vs the reference's tableaux (golden) and the new
Gauss-Legendre / real-Schur known answers (CPU)."""

import numpy as np
import pytest

from paper_2403_08084_b200 import tableaux as tb


@pytest.mark.parametrize("s", [1, 2, 3, 4, 5])
def test_radau_matches_reference(golden, s):
    t = tb.radau_iia(s)
    np.testing.assert_allclose(t.A, golden[f"tab_radau{s}_A"], rtol=0, atol=5e-15)
    np.testing.assert_allclose(t.b, golden[f"tab_radau{s}_b"], rtol=0, atol=5e-15)
    np.testing.assert_array_equal(t.c[-1], 1.0)
    np.testing.assert_allclose(t.c, golden[f"tab_radau{s}_c"], rtol=0, atol=1e-15)
    assert t.stiffly_accurate and t.invertible


@pytest.mark.parametrize("name,ctor", [("lobatto2", lambda: tb.lobatto_iiic(2)),
                                       ("lobatto3", lambda: tb.lobatto_iiic(3)),
                                       ("alexander", tb.alexander_dirk),
                                       ("wsodirk", tb.wsodirk433)])
def test_fixed_tableaux_match_reference(golden, name, ctor):
    t = ctor()
    for f in ("A", "b", "c"):
        np.testing.assert_allclose(getattr(t, f), golden[f"tab_{name}_{f}"], rtol=0, atol=3e-15)


def test_alexander_gamma():
    # tests/test_tableaux.py:110-114 pins gamma
    assert tb.alexander_dirk().A[0, 0] == pytest.approx(0.435866521508459, abs=1e-14)
    assert tb.alexander_dirk().lower_triangular and tb.alexander_dirk().stiffly_accurate


@pytest.mark.parametrize("s", [1, 2, 3, 4, 5])
def test_gauss_legendre_order_conditions(s):
    t = tb.gauss_legendre(s)
    b_res, st_res = tb.order_condition_residuals(t, 2 * s, s)
    assert b_res.max() < 1e-13 and st_res.max() < 1e-13
    assert not t.stiffly_accurate and t.invertible
    if s == 1:  # implicit midpoint
        assert t.A[0, 0] == pytest.approx(0.5) and t.c[0] == pytest.approx(0.5)


def test_gauss_spec_names():
    assert tb.from_spec("gauss-legendre:4").s == 4
    with pytest.raises(tb.UnsupportedStageCountError):
        tb.from_spec("gauss:2")  # the bare family stays unknown (tests/test_tableaux.py:289-290)


@pytest.mark.parametrize("tab", [tb.gauss_legendre(4), tb.gauss_legendre(3), tb.radau_iia(3),
                                 tb.radau_iia(5), tb.gauss_legendre(2)], ids=lambda t: t.name)
def test_real_schur(tab):
    sd = tb.real_schur(tab.A)
    assert np.abs(sd.Q @ sd.T @ sd.Q.T - tab.A).max() < 1e-14
    assert np.abs(sd.Q.T @ sd.Q - np.eye(tab.s)).max() < 1e-14
    ev = np.sort_complex(np.linalg.eigvals(tab.A))
    got = []
    for st, sz in sd.blocks:
        B = sd.T[st:st + sz, st:st + sz]
        if sz == 2:
            assert B[0, 0] == B[1, 1] and B[0, 1] * B[1, 0] < 0
        got.extend(np.linalg.eigvals(B))
    np.testing.assert_allclose(np.sort_complex(np.array(got)), ev, atol=1e-13)


def test_gl4_has_two_complex_pairs():
    sd = tb.real_schur(tb.gauss_legendre(4).A)
    assert [sz for _, sz in sd.blocks] == [2, 2]


def test_ldu_and_split_round_trip():
    for t in (tb.radau_iia(3), tb.lobatto_iiic(3), tb.gauss_legendre(3)):
        f = tb.ldu_factor(t)
        np.testing.assert_allclose(f.reconstruct(), t.A, atol=1e-14)
        np.testing.assert_allclose(tb.additive_split(t).reconstruct(), t.A, atol=0)


def test_csv_round_format():
    text = tb.to_csv(tb.lobatto_iiic(2))
    assert text.splitlines()[0] == "stage,c,a_1,a_2"
    assert text.splitlines()[-1].startswith("b,,")
