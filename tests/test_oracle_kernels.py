"""Pin the CPU oracle against the reference's literal known answers.

Mirrors reference tests/test_kernels.cpp, test_locations.cpp and the
tridiagonal KAT of test_krylov.cpp:113-139. CPU only.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from tests import dense_mirror as DM


def test_rng_known_answers():
    # C++ [rand.predef]: the 10000th output of a default-seeded mt19937_64
    assert O.lib().orc_mt19937_64_nth(5489, 10000) == 9981545732273789042
    # SplitMix64 reference output for state 0
    assert O.splitmix64(0) == 0xE220A8397B1DCDAF


def test_probe_streams_are_keyed():
    a1, a2 = O.probe_gaussian(7, 3, 5, 11)
    b1, b2 = O.probe_gaussian(7, 3, 5, 11)
    assert np.array_equal(a1, b1) and np.array_equal(a2, b2)
    c1, _ = O.probe_gaussian(7, 4, 5, 11)
    assert not np.array_equal(a1, c1)
    z = O.probe_rademacher(1, 2, 1000)
    assert set(np.unique(z)) == {-1.0, 1.0}


def test_matern_literal_values():  # test_kernels.cpp:12-21
    s3, s5 = math.sqrt(3.0), math.sqrt(5.0)
    assert O.matern(0.5, 1.5, 2.0, 0.5) == pytest.approx(2.0 * (1.0 + s3) * math.exp(-s3), rel=1e-14)
    assert O.matern(0.0, 1.5, 1.7, 0.2) == pytest.approx(1.7, rel=1e-15)
    assert O.matern(0.3, 0.5, 1.0, 0.3) == pytest.approx(math.exp(-1.0), rel=1e-14)
    assert O.matern(0.2, 2.5, 1.0, 0.2) == pytest.approx((1.0 + s5 + 5.0 / 3.0) * math.exp(-s5), rel=1e-14)


def test_matern_random_and_derivative():  # test_kernels.cpp:23-50
    rng = np.random.default_rng(7)
    for _ in range(200):
        d, s1, rho = 2.0 * rng.random(), 0.1 + 2.0 * rng.random(), 0.05 + 0.5 * rng.random()
        for nu in (0.5, 1.5, 2.5):
            assert O.matern(d, nu, s1, rho) == pytest.approx(float(DM.matern_ref(d, nu, s1, rho)), rel=1e-13)
    for nu in (0.5, 1.5, 2.5):
        for d in (0.01, 0.1, 0.4, 1.3):
            for rho in (0.05, 0.2, 0.7):
                h = 1e-6 * rho
                fd = (O.matern(d, nu, 1.3, rho + h) - O.matern(d, nu, 1.3, rho - h)) / (2 * h)
                assert O.matern_drho(d, nu, 1.3, rho) == pytest.approx(fd, rel=1e-6)


def test_taper_literal_values():  # test_kernels.cpp:52-69
    assert O.taper_value(0.5, 1, 1.0) == pytest.approx(0.1875, rel=1e-15)
    assert O.taper_value(0.0, 1, 1.0) == pytest.approx(1.0, rel=1e-15)
    assert O.taper_value(1.0, 1, 1.0) == 0.0
    assert O.taper_value(2.0, 1, 1.0) == 0.0
    assert O.taper_value(0.5, 2, 1.0) == pytest.approx(0.5 ** 6 * (1 + 3 + 35 * 0.25 / 3), rel=1e-14)
    assert O.taper_value(1.0, 2, 1.0) == 0.0
    for d in np.arange(0.0, 1.0, 0.01):
        for fam in (1, 2):
            assert O.taper_value(d, fam, 1.0) == pytest.approx(float(DM.wendland_ref(d, 1.0, fam)), rel=1e-12, abs=1e-300)


def test_range_calibration():  # test_kernels.cpp:71-77
    rho = O.rho_for_correlation_at(0.2, 0.05, 1.5)
    assert rho == pytest.approx(0.0741, rel=0.02)
    assert O.matern(0.2, 1.5, 1.0, rho) == pytest.approx(0.05, rel=1e-6)
    assert O.effective_range(rho, 1.5) == pytest.approx(0.2, rel=1e-4)


def test_uniform_locations():  # test_locations.cpp:14-22
    a = O.uniform_locations(200, 3, 11)
    b = O.uniform_locations(200, 3, 11)
    c = O.uniform_locations(200, 3, 12)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    assert a.min() >= 0.0 and a.max() <= 1.0


def test_taper_pattern_equals_brute_force():  # test_locations.cpp:24-45
    locs = O.uniform_locations(120, 2, 21)
    gamma = 0.15
    ptr, idx, val = O.taper_pattern(locs, gamma)
    D = DM.pairwise(locs, locs)
    expected = {(i, i) for i in range(120)} | {(i, j) for i in range(120) for j in range(120) if i != j and D[i, j] < gamma}
    got = set()
    for i in range(120):
        cols = idx[ptr[i]:ptr[i + 1]]
        assert np.all(np.diff(cols) > 0)  # sorted, unique
        for p in range(ptr[i], ptr[i + 1]):
            got.add((i, int(idx[p])))
            assert val[p] == pytest.approx(D[i, idx[p]], rel=1e-14, abs=1e-300)
    assert got == expected


def test_cross_pattern():  # test_locations.cpp:47-66
    rows = O.uniform_locations(60, 2, 31)
    cols = O.uniform_locations(40, 2, 32)
    ptr, idx, val = O.cross_taper_pattern(rows, cols, 0.2)
    D = DM.pairwise(rows, cols)
    assert len(ptr) == 61
    assert np.all(val < 0.2)
    assert len(idx) == int((D < 0.2).sum())
    for i in range(60):
        np.testing.assert_allclose(val[ptr[i]:ptr[i + 1]], D[i, idx[ptr[i]:ptr[i + 1]]], rtol=1e-14)


def test_gamma_for_row_nnz():  # locations.cpp:192-195
    assert O.gamma_for_avg_row_nnz(10000, 30.0) == pytest.approx(math.sqrt(30.0 / (10000 * math.pi)))


def test_tridiag_quadrature_known_answer():  # test_krylov.cpp:113-139
    d = np.array([2.0, 2.5, 3.0, 2.2, 1.8])
    e = np.array([0.4, 0.3, 0.5, 0.2])
    T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    w, V = np.linalg.eigh(T)
    want = float((V[0, :] ** 2 * np.log(w)).sum())
    assert O.tridiag_log_quadrature(d, e) == pytest.approx(want, rel=1e-12)
    assert O.tridiag_log_quadrature(np.zeros(0), np.zeros(0)) == 0.0
    with pytest.raises(O.NumericalError):
        O.tridiag_log_quadrature(np.array([-1.0]), np.zeros(0))


def test_tridiag_quadrature_random():
    rng = np.random.default_rng(3)
    for k in (1, 2, 7, 40, 120):
        d = 1.0 + 3.0 * rng.random(k)
        e = 0.5 * rng.random(max(k - 1, 0))
        T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
        w, V = np.linalg.eigh(T)
        want = float((V[0, :] ** 2 * np.log(w)).sum())
        assert O.tridiag_log_quadrature(d, e) == pytest.approx(want, rel=1e-11, abs=1e-13)


def test_select_random_and_kmeanspp():
    locs = O.uniform_locations(500, 2, 5)
    ind = O.select_random(locs, 20, 9)
    assert ind.shape == (20, 2)
    rows = {tuple(r) for r in locs}
    assert all(tuple(r) in rows for r in ind)
    assert len({tuple(r) for r in ind}) == 20
    km = O.select_kmeanspp(locs, 25, 9)
    assert all(tuple(r) in rows for r in km)
    assert len({tuple(r) for r in km}) == 25
    assert np.array_equal(km, O.select_kmeanspp(locs, 25, 9))
