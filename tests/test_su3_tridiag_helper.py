"""Pins for the test-side 40-digit construction of the GPU's general spin-one factor (tests/su3_tridiag_mp.py,
reading R20) that the low-τ GPU tests compare against: it must be exp(−iH) at large τ (a second-order splitting) and,
with no U/V coefficients, reproduce the paper's own factor of Eq. lie_trotter_4 — the oracle's four-operator
exponentiator — at every τ.  No GPU needed."""
import numpy as np
import scipy.linalg as sl

import workloads as W
from su3_tridiag_mp import H8, tridiag_factor


def test_helper_is_exp_at_large_tau():
    for x in W.random_exponent_args_su3(8, 0.5, seed=61):
        assert np.abs(tridiag_factor(x, 24)[1] - sl.expm(-1j * H8(x))).max() < 1e-15


def test_helper_is_second_order():
    x = W.random_exponent_args_su3(1, 0.2, seed=62)[0]
    errs = [np.abs(tridiag_factor(s * x, 0)[1] - sl.expm(-1j * H8(s * x))).max() for s in (1.0, 0.5, 0.25)]
    assert 6.5 < errs[0] / errs[1] < 9.5 and 6.5 < errs[1] / errs[2] < 9.5, errs


def test_helper_reduces_to_paper_factor(orc):
    """u = v = 0: the tridiagonalising similarity is the paper's diagonal phase R_φ (up to a global phase), so the
    factor is Eq. lie_trotter_4's T exactly (oracle, four-operator exponentiator), also at low τ."""
    for x in W.random_exponent_args(6, 1.0, seed=63):
        for tau in (0, 3):
            ref = orc.exponentiate("one", x[None], "lie_trotter", tau)[0]
            assert np.abs(tridiag_factor(np.r_[x, np.zeros(4)], tau)[1] - ref).max() < 1e-15
