"""CPU-side checks of the product boundary: the C-ABI library loads, exports every
symbol include/fsa_b200.h declares, and its host-side input generators reproduce
the reference's RNG streams (checked against the oracle). No GPU compute here."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import oracle as O
from paper_2405_14492_b200 import fsa

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "fsa_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int64_t|int|void|double)\s+(fsa_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(fsa.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 40
    missing = [nm for nm in names if not hasattr(L, nm)]
    assert not missing, missing
    assert fsa.lib().fsa_version() == 1


def test_generators_match_reference_streams():
    a = fsa.uniform_locations(500, 2, 11)
    assert np.array_equal(a, O.uniform_locations(500, 2, 11))
    assert np.array_equal(fsa.select_random(a, 40, 3), O.select_random(a, 40, 3))
    assert np.array_equal(fsa.select_kmeanspp(a, 25, 9), O.select_kmeanspp(a, 25, 9))
    assert fsa.gamma_for_avg_row_nnz(10000, 30.0) == O.gamma_for_avg_row_nnz(10000, 30.0)
    for i in (0, 1, 7):
        e1, e2 = fsa.probe_gaussian(123, i, 13, 101)
        o1, o2 = O.probe_gaussian(123, i, 13, 101)
        assert np.array_equal(e1, o1) and np.array_equal(e2, o2)


def test_tridiag_quadrature_host():
    d = np.array([2.0, 2.5, 3.0, 2.2, 1.8])
    e = np.array([0.4, 0.3, 0.5, 0.2])
    T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    w, V = np.linalg.eigh(T)
    assert fsa.tridiag_log_quadrature(d, e) == pytest.approx(float((V[0] ** 2 * np.log(w)).sum()), rel=1e-12)
    with pytest.raises(fsa.NumericalError):
        fsa.tridiag_log_quadrature(np.array([-1.0]), np.zeros(0))


def test_rff_and_blobs_are_seeded():
    c = fsa.uniform_locations(300, 2, 1)
    y1 = fsa.simulate_rff(c, 1.5, 1.0, 0.1, 0.1, 128, 7)
    y2 = fsa.simulate_rff(c, 1.5, 1.0, 0.1, 0.1, 128, 7)
    assert np.array_equal(y1, y2) and np.isfinite(y1).all() and 0.3 < y1.var() < 3.0
    b = fsa.blob_locations(1000, 2, 50, 0.01, 3)
    assert b.min() >= 0.0 and b.max() <= 1.0


def test_invalid_arguments_raise_without_gpu():
    with pytest.raises(ValueError):
        fsa.uniform_locations(0, 2, 1)
    with pytest.raises(ValueError):
        fsa.select_random(fsa.uniform_locations(10, 2, 1), 20, 1)
