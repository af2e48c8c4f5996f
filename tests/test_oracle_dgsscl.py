"""Pins of the oracle's real Gram-Schmidt orthogonalization dgsscl (NEXT-4,
Alg SM8.1 / Eq. (DGS); reading R#39) against things
other than itself: exact rational evaluation of Eq. (DGS) on dyadic inputs,
the parallel and orthogonal special cases, scale equivariance, and the
orthogonality of the result in the regime it exists for (||g_q|| << ||g_p||)."""
from fractions import Fraction

import numpy as np
import pytest

import oracle as O


def _dgs_exact(gp, gq, ep, fp, eq, fq, a21):
    """Eq. (DGS) in exact arithmetic with psi = a21 (fq / fp) exact."""
    psi = Fraction(a21) * Fraction(fq) / Fraction(fp)
    two = Fraction(2)
    return [(Fraction(y) / two ** int(eq) - psi * Fraction(x) / two ** int(ep)) * two ** int(eq)
            for x, y in zip(gp, gq)]


def test_worked_example():
    gp = np.array([4.0, -2.0, 6.0])
    gq = np.array([3.0, 5.0, -1.0])
    out = O.dgsscl(gp, gq, 2.0, 1.0, 1.0, 1.5, 0.25)  # psi = 0.375
    assert np.array_equal(out, [2.25, 5.375, -2.125])


@pytest.mark.parametrize("seed", range(6))
def test_exact_on_dyadic_inputs(seed):
    # small-integer columns and dyadic (f, a21) with f_q / f_p exact: every
    # operation of Alg SM8.1 is exact, so the result is Eq. (DGS) exactly
    rng = np.random.default_rng(seed)
    m = 200
    ep, eq = float(rng.integers(-400, 400)), float(rng.integers(-400, 400))
    # x = g_p 2^-e_p and y = g_q 2^-e_q within 2^+-8 of each other: fma exact
    gp = rng.integers(-64, 65, m).astype(np.float64) * 2.0 ** (int(ep) + int(rng.integers(-4, 4)))
    gq = rng.integers(-64, 65, m).astype(np.float64) * 2.0 ** (int(eq) + int(rng.integers(-4, 4)))
    fp = 1.0
    fq = float(rng.integers(2, 8)) / 4.0 + 1.0  # 1.5, 1.75, ... exact quotient by fp = 1
    fq = min(fq, 1.75)
    a21 = float(rng.integers(-8, 9)) / 16.0
    out = O.dgsscl(gp, gq, ep, fp, eq, fq, a21)
    ref = _dgs_exact(gp, gq, ep, fp, eq, fq, a21)
    assert all(Fraction(o) == r for o, r in zip(out, ref))


def test_parallel_columns_vanish_and_orthogonal_ones_stay():
    rng = np.random.default_rng(1)
    gp = rng.standard_normal(300)
    # g_q = 2^k g_p: same f, e shifted by k, a21' = 1 -> psi = 1 -> g_q' = 0 exactly
    for k in (-7, 0, 12):
        out = O.dgsscl(gp, gp * 2.0 ** k, 3.0, 1.25, 3.0 + k, 1.25, 1.0)
        assert np.array_equal(out, np.zeros(300))
    # a21' = 0: g_q unchanged bit for bit
    gq = rng.standard_normal(300) * 2.0 ** rng.integers(-10, 10, 300)
    assert np.array_equal(O.dgsscl(gp, gq, 0.0, 1.1, 4.0, 1.3, 0.0), gq)


def test_scale_equivariance():
    rng = np.random.default_rng(2)
    gp = rng.standard_normal(257)
    gq = rng.standard_normal(257)
    base = O.dgsscl(gp, gq, 4.0, 1.2, 4.0, 1.6, -0.3)
    for k in (-500, -60, 77, 600):
        # g_q -> 2^k g_q (e_q + k): result scales by 2^k exactly
        assert np.array_equal(O.dgsscl(gp, gq * 2.0 ** k, 4.0, 1.2, 4.0 + k, 1.6, -0.3),
                              base * 2.0 ** k)
        # g_p -> 2^k g_p (e_p + k): result unchanged
        assert np.array_equal(O.dgsscl(gp * 2.0 ** k, gq, 4.0 + k, 1.2, 4.0, 1.6, -0.3), base)


@pytest.mark.parametrize("kp,kq", [(0, 0), (900, -900), (-500, 400), (1000, -1000)])
def test_orthogonalizes_when_norms_differ(kp, kq):
    # the regime of P:1369-1378: ||g_q|| << ||g_p|| (tan phi would underflow)
    rng = np.random.default_rng(abs(kp - kq) + 5)
    m = 400
    u = rng.standard_normal(m)
    w = rng.standard_normal(m) + 0.3 * u  # correlated with u
    gp, gq = u * 2.0 ** kp, w * 2.0 ** kq
    # the true norms (of the unscaled u, w, shifted) and the exact cosine
    nu = float(np.sqrt(float(sum(Fraction(float(v)) ** 2 for v in u))))
    nw = float(np.sqrt(float(sum(Fraction(float(v)) ** 2 for v in w))))
    mu_, exu = np.frexp(nu)
    mw_, exw = np.frexp(nw)
    ep, fp = float(exu - 1 + kp), float(mu_ * 2)
    eq, fq = float(exw - 1 + kq), float(mw_ * 2)
    dot = sum(Fraction(float(a)) * Fraction(float(b)) for a, b in zip(u, w))
    a21 = float(dot / (Fraction(nu) * Fraction(nw)))
    out = O.dgsscl(gp, gq, ep, fp, eq, fq, a21)
    assert np.all(np.isfinite(out))
    # cosine of the angle between g_q' and g_p (computed on the unscaled values)
    o = out * 2.0 ** -kq
    c = float(sum(Fraction(float(a)) * Fraction(float(b)) for a, b in zip(u, o)))
    no = float(np.sqrt(float(sum(Fraction(float(v)) ** 2 for v in o))))
    assert abs(c) / (nu * no) <= 8 * m * 2.0 ** -53
