"""Pins for the single-precision EVD of the oracle (orc_evd2_one_f32; Alg 2.2 /
SM2.1 converted to binary32 as P:709-717 prescribes: omega = FLT_MAX,
fl(sqrt(omega)) = 1.844674297E+19, mu_check = FLT_TRUE_MIN, eta = FLT_MAX_EXP - 4).

Expected values come from the paper's constants, closed forms, exact rational
arithmetic and 60-digit mpmath -- never from the oracle itself.  CPU only.
"""
import math
from fractions import Fraction

import mpmath
import numpy as np
import pytest

import oracle as O

F = np.float32
EPS = 2.0 ** -24
FMAX = float(np.finfo(np.float32).max)
MU = float(np.finfo(np.float32).smallest_subnormal)  # 2^-149
SQRT_OMEGA_F = float.fromhex("0x1.fffffep+63")


def f32bits(x):
    return np.array([x], dtype=np.float32).view(np.uint32)[0]


def test_constants_of_the_single_precision_conversion():
    # P:712 prints fl(sqrt(omega)) = 1.844674297E+19
    assert float(F(1.844674297e19)) == SQRT_OMEGA_F
    assert float(F(math.sqrt(FMAX))) == SQRT_OMEGA_F
    # fma(fl(sqrt w), fl(sqrt w), 1) is finite in binary32 (no overflow in Eq. tan2 / jactan)
    assert Fraction(SQRT_OMEGA_F) ** 2 + 1 < Fraction(FMAX)
    assert MU == 2.0 ** -149 and FMAX == float.fromhex("0x1.fffffep+127")


@pytest.mark.parametrize("a11,a22,re,im,expect", [
    (1.0, 1.0, 0.0, 0.0, 124),       # eta - lg 1
    (3.0, 1.0, 0.0, 0.0, 123),       # floor(lg 3) = 1
    (FMAX / 8, FMAX / 8, FMAX / 8, FMAX / 8, 0),   # lg(FMAX/8) = 124
    (0.0, 0.0, MU, 0.0, 124 + 149),  # a single mu_check entry
    (FMAX, 0.0, 0.0, 0.0, -3),       # lg FLT_MAX = 127
])
def test_zeta_examples(a11, a22, re, im, expect):
    assert O.evd2_one_f32(True, a11, a22, re, im)["zeta"] == expect


def test_zeta_zero_matrix_sentinel():
    assert O.zeta_f32(0.0, 0.0, 0.0, 0.0) == FMAX
    assert O.evd2_one_f32(True, 0.0, 0.0, 0.0, 0.0)["zeta"] == O.ZETA_ZERO


def test_hypot_examples():
    assert O.hypot_f32(3.0, 4.0) == 5.0
    assert O.hypot_f32(MU, MU) == MU          # sqrt2 * mu rounds back to mu
    assert O.hypot_f32(0.0, 0.0) == 0.0       # max(0/0, 0) = 0
    x = 1.5
    assert O.hypot_f32(x, x) == float(F(F(math.sqrt(2.0)) * F(x)))


def test_diagonal_gives_identity():
    rng = np.random.default_rng(3)
    for _ in range(500):
        a11, a22 = (float(F(v)) for v in rng.standard_normal(2) * 2.0 ** rng.integers(-60, 60, 2))
        r = O.evd2_one_f32(True, a11, a22, 0.0, 0.0)
        assert r["cos"] == 1.0 and r["sin_re"] == 0.0 and r["sin_im"] == 0.0
        assert (r["lam1"], r["lam2"]) == (F(a11), F(a22))


def test_zero_diagonal_unit_offdiagonal():
    r = O.evd2_one_f32(False, 0.0, 0.0, 1.0)
    assert r["lam1"] == 1.0 and r["lam2"] == -1.0
    c = F(F(1.0) / F(math.sqrt(2.0)))
    assert r["cos"] == c and r["sin_re"] == c  # tan = 1: sin = 1/sec = cos


@pytest.mark.parametrize("sgn", [1.0, -1.0])
def test_evil_matrix_single_precision_analogue_of_eq51(sgn):
    # a11 = a22 = FLT_MAX/8, a21 = mu (1 +- i): zeta = 0, |a21| = mu, a = 0 so
    # tan 2phi clamps to fl(sqrt w) and tan phi rounds to 1; e^{ia} = 1 +- i
    # (Remark 2.4's pathology in binary32)
    r = O.evd2_one_f32(True, FMAX / 8, FMAX / 8, MU, sgn * MU, O.EVD_TAN)
    assert r["zeta"] == 0
    assert r["cos"] == F(F(1.0) / F(math.sqrt(2.0)))
    assert r["sin_re"] == 1.0 and r["sin_im"] == sgn
    assert r["lam1"] == F(FMAX / 8) and r["lam2"] == F(FMAX / 8)


def test_real_equals_complex_with_zero_imag():
    rng = np.random.default_rng(4)
    for _ in range(3000):
        a = [float(F(v)) for v in rng.standard_normal(3) * 2.0 ** rng.integers(-40, 40, 3)]
        for fl in (0, O.EVD_TAN):
            rr = O.evd2_one_f32(False, *a, flags=fl)
            rc = O.evd2_one_f32(True, *a, 0.0, flags=fl)
            for k in ("lam1", "lam2", "cos", "sin_re"):
                assert f32bits(rr[k]) == f32bits(rc[k]), (a, k)


def _givens_f32(n, cplx, seed):
    """A = U(phi, alpha) diag(lam) U^H assembled exactly and rounded to binary32."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        t = Fraction(float(rng.random())) * Fraction(2) ** int(rng.integers(-20, 1))
        lam = [Fraction(float(rng.standard_normal())) * Fraction(2) ** int(rng.integers(-30, 30))
               for _ in range(2)]
        al = rng.random() * 2 * math.pi if cplx else (0.0 if rng.random() < 0.5 else math.pi)
        ca, sa = Fraction(math.cos(al)), Fraction(math.sin(al))
        c2 = 1 / (1 + t * t)
        a11 = c2 * (lam[0] + lam[1] * t * t)
        a22 = c2 * (lam[0] * t * t + lam[1])
        off = c2 * t * (lam[0] - lam[1])
        out.append(tuple(float(F(float(v))) for v in (a11, a22, off * ca, off * sa)))
    return out


def _exact_scaled(a11, a22, re, im, z):
    s = mpmath.mpf(2) ** z
    return (mpmath.mpf(a11) * s, mpmath.mpf(a22) * s, mpmath.mpf(re) * s, mpmath.mpf(im) * s)


@pytest.mark.parametrize("cplx", [False, True])
def test_prop22_bounds_hold_in_single_precision(cplx):
    # "the relative error bounds in Prop 2.2 still hold" with eps = 2^-24:
    # cos phi < 8.000002 eps (R) / 14.000006 eps (C); tan phi < 5.500001 / 11.500004
    # eps; eigenvalues normwise <= 8 eps (SM7.1)
    mpmath.mp.dps = 60
    tb, cb = (11.500004, 14.000006) if cplx else (5.500001, 8.000002)
    worst = dict(tan=0.0, cos=0.0, lam=0.0)
    for a11, a22, re, im in _givens_f32(1500, cplx, 51 + int(cplx)):
        r = O.evd2_one_f32(cplx, a11, a22, re, im, O.EVD_TAN | O.EVD_NOBACKSCALE)
        s11, s22, sre, sim = _exact_scaled(a11, a22, re, im, r["zeta"])
        ab = mpmath.sqrt(sre ** 2 + sim ** 2)
        a = s11 - s22
        if ab == 0 or a == 0:
            continue
        t2 = 2 * ab / abs(a)
        t = t2 / (1 + mpmath.sqrt(1 + t2 * t2))
        c = 1 / mpmath.sqrt(1 + t * t)
        if t < mpmath.mpf(2) ** -120:
            continue
        worst["cos"] = max(worst["cos"], float(abs(mpmath.mpf(float(r["cos"])) / c - 1)) / EPS)
        et = mpmath.sqrt(mpmath.mpf(float(r["sin_re"])) ** 2 + mpmath.mpf(float(r["sin_im"])) ** 2)
        worst["tan"] = max(worst["tan"], float(abs(et / t - 1)) / EPS)
        mid, rad = (s11 + s22) / 2, mpmath.sqrt((a / 2) ** 2 + ab ** 2)
        ex = sorted([mid + rad, mid - rad])
        got = sorted([mpmath.mpf(float(r["lam1"])), mpmath.mpf(float(r["lam2"]))])
        nrm = mpmath.sqrt(ex[0] ** 2 + ex[1] ** 2)
        worst["lam"] = max(worst["lam"], float(mpmath.sqrt((got[0] - ex[0]) ** 2 +
                                                           (got[1] - ex[1]) ** 2) / nrm) / EPS)
    assert worst["cos"] < cb, worst
    assert worst["lam"] <= 8.0, worst
    assert worst["tan"] < tb + (4.000001 + 1e-3 if cplx else 0.0), worst


@pytest.mark.parametrize("cplx", [False, True])
def test_trace_and_determinant_invariants_f32(cplx):
    mpmath.mp.dps = 60
    for a11, a22, re, im in _givens_f32(600, cplx, 61 + int(cplx)):
        r = O.evd2_one_f32(cplx, a11, a22, re, im, O.EVD_NOBACKSCALE)
        s11, s22, sre, sim = _exact_scaled(a11, a22, re, im, r["zeta"])
        l1, l2 = mpmath.mpf(float(r["lam1"])), mpmath.mpf(float(r["lam2"]))
        scale = abs(l1) + abs(l2)
        if scale == 0:
            continue
        assert abs((l1 + l2) - (s11 + s22)) <= 8 * EPS * scale
        det = s11 * s22 - (sre ** 2 + sim ** 2)
        assert abs(l1 * l2 - det) <= 16 * EPS * scale ** 2


def test_no_overflow_near_flt_max_and_subnormals():
    rng = np.random.default_rng(9)
    vals = [FMAX, -FMAX, FMAX / 2, MU, -MU, 0.0, 2.0 ** -126, 1.0]
    for _ in range(3000):
        a = [float(rng.choice(vals)) for _ in range(4)]
        r = O.evd2_one_f32(True, *a, flags=O.EVD_NOBACKSCALE)
        for k in ("lam1", "lam2", "cos", "sin_re", "sin_im"):
            assert math.isfinite(r[k]), (a, r)
        assert 0.0 < r["cos"] <= 1.0
    r = O.evd2_one_f32(True, FMAX, FMAX, FMAX, FMAX)   # R#7: backscaled lambda may overflow
    assert r["lam1"] == math.inf
    r = O.evd2_one_f32(True, FMAX, FMAX, FMAX, FMAX, O.EVD_NOBACKSCALE)
    assert math.isfinite(r["lam1"]) and r["zeta"] == -3


def test_single_agrees_with_double_to_single_precision():
    # the same algorithm in binary64 on the same (float-representable) inputs:
    # cos and the eigenvalues agree to a few units of 2^-24
    rng = np.random.default_rng(12)
    n = 4000
    a = (rng.standard_normal((4, n)) * 2.0 ** rng.integers(-30, 30, (4, n))).astype(np.float32)
    R32 = O.evd2_batched_f32(a[0], a[1], a[2], a[3])
    R64 = O.evd2_batched(a[0].astype(np.float64), a[1].astype(np.float64),
                         a[2].astype(np.float64), a[3].astype(np.float64))
    assert np.all(np.abs(R32["cos"] - R64["cos"]) <= 16 * EPS)
    nrm = np.hypot(R64["lam1"], R64["lam2"])
    err = np.hypot(R32["lam1"] - R64["lam1"], R32["lam2"] - R64["lam2"])
    assert np.all(err <= 16 * EPS * nrm)


def test_batched_equals_one_by_one_and_perm_words_f32():
    rng = np.random.default_rng(14)
    n = 1000
    a = (rng.standard_normal((4, n)) * 2.0 ** rng.integers(-10, 10, (4, n))).astype(np.float32)
    R = O.evd2_batched_f32(*a)
    for l in range(0, n, 37):
        o = O.evd2_one_f32(True, *(a[k][l] for k in range(4)))
        for k in ("lam1", "lam2", "cos", "sin_re", "sin_im"):
            assert f32bits(o[k]) == R[k].view(np.uint32)[l]
        assert o["zeta"] == R["zeta"][l]
        assert ((R["perm"][l // 32] >> (l % 32)) & 1) == o["perm"]
