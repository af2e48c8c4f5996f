"""Pins for the EVD part of the oracle (oracle/jsvd_oracle.c, Alg 2.2 / SM2.1).

Every expected value here comes from the paper's worked examples, closed forms,
exact rational arithmetic (fractions.Fraction) or 60-digit mpmath -- never from
the oracle itself and never from the CUDA path.  CPU only.
"""
import math
import struct
from fractions import Fraction

import mpmath
import numpy as np
import pytest

import oracle as O
import synth

EPS = 2.0 ** -53
OMEGA = np.finfo(np.float64).max
MU = 5e-324  # mu-check, smallest positive subnormal
SQRT_OMEGA = float.fromhex("0x1.fffffffffffffp+511")


def bits(x):
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def floor_lg(x):
    """floor(lg|x|) for finite nonzero x, from the exact binary decomposition."""
    m, e = math.frexp(abs(x))
    return e - 1


# ---------------------------------------------------------------- constants
def test_sqrt_omega_constant():
    # P:736 prints fl(sqrt(omega)) = 1.34078079299425956E+154
    assert SQRT_OMEGA == float("1.34078079299425956E+154")
    assert SQRT_OMEGA == math.sqrt(OMEGA)
    # fma(fl(sqrt w), fl(sqrt w), 1) cannot overflow
    assert math.isfinite(float(Fraction(SQRT_OMEGA) ** 2 + 1))


# ---------------------------------------------------------------- zeta, Eq. (z)
@pytest.mark.parametrize("a11,a22,re,im,expect", [
    (1.0, 1.0, 0.0, 0.0, 1020),            # eta - 0
    (3.0, 1.0, 0.0, 0.0, 1019),            # floor(lg 3) = 1
    (OMEGA / 8, -OMEGA / 8, OMEGA / 8, -OMEGA / 8, 0),
    (0.0, 0.0, MU, 0.0, 2094),             # 1020 + 1074
    (OMEGA, 1.0, 0.0, 0.0, -3),            # 1020 - 1023
])
def test_zeta_examples(a11, a22, re, im, expect):
    assert O.zeta(a11, a22, re, im) == expect
    assert O.evd2_one(True, a11, a22, re, im)["zeta"] == expect


def test_zeta_zero_matrix_sentinel():
    assert O.zeta(0.0, 0.0, 0.0, 0.0) == OMEGA  # zeta = omega
    r = O.evd2_one(True, 0.0, 0.0, 0.0, 0.0)
    assert r["zeta"] == O.ZETA_ZERO
    assert (r["lam1"], r["lam2"], r["cos"], r["sin_re"], r["sin_im"]) == (0.0, 0.0, 1.0, 0.0, 0.0)


def test_zeta_matches_exact_floor_lg_random():
    rng = np.random.default_rng(1)
    for _ in range(2000):
        v = [float(x) for x in rng.standard_normal(4) * 2.0 ** rng.integers(-1070, 1020, 4)]
        for k in range(4):
            if rng.random() < 0.2:
                v[k] = 0.0
        nz = [x for x in v if x != 0.0]
        expect = min(1020 - floor_lg(x) for x in nz) if nz else O.ZETA_ZERO
        assert O.evd2_one(True, *v)["zeta"] == expect


# ---------------------------------------------------------------- hypot, Alg 2.1
def test_hypot_examples():
    assert O.hypot(3.0, 4.0) == 5.0
    assert O.hypot(-3.0, 4.0) == 5.0
    assert O.hypot(0.0, 0.0) == 0.0
    assert O.hypot(MU, MU) == MU  # Remark 2.4: mu-check is in Psi
    rng = np.random.default_rng(2)
    for x in rng.standard_normal(500) * 2.0 ** rng.integers(-1000, 1000, 500):
        # Remark 2.4: fl(hypot(x,x)) = fl(fl(sqrt2)|x|) for normal x
        assert O.hypot(x, x) == math.sqrt(2.0) * abs(x)


def test_hypot_lemma21_bound():
    # Lemma 2.1: relative error within delta_2^{+-}
    mpmath.mp.dps = 60
    eps = mpmath.mpf(2) ** -53
    dp = (1 + eps) ** mpmath.mpf(2.5) * mpmath.sqrt(1 + eps * (2 + eps) / 2)
    dm = (1 - eps) ** mpmath.mpf(2.5) * mpmath.sqrt(1 - eps * (2 - eps) / 2)
    rng = np.random.default_rng(3)
    for _ in range(3000):
        x, y = rng.standard_normal(2) * 2.0 ** rng.integers(-500, 500, 2)
        h = mpmath.sqrt(mpmath.mpf(x) ** 2 + mpmath.mpf(y) ** 2)
        r = mpmath.mpf(O.hypot(x, y)) / h
        assert dm < r < dp


# ---------------------------------------------------------------- worked examples
def test_polar_3_4i():
    # Eq. (zpolar) on 3+4i: cos a = 0.6, sin a = 0.8; a11 = a22 = 0 => tan phi = 1
    r = O.evd2_one(True, 0.0, 0.0, 3.0, 4.0, O.EVD_TAN)
    assert r["sin_re"] == 0.6 and r["sin_im"] == 0.8
    assert r["cos"] == 1.0 / math.sqrt(2.0)
    assert (r["lam1"], r["lam2"]) == (5.0, -5.0)


def test_diagonal_gives_identity():
    # a21 = 0 -> identity eigenvectors, lambda = (a11, a22) exactly
    rng = np.random.default_rng(4)
    for a11, a22 in rng.standard_normal((500, 2)) * 2.0 ** rng.integers(-900, 900, (500, 2)):
        for cplx in (False, True):
            r = O.evd2_one(cplx, a11, a22, 0.0, 0.0)
            assert r["cos"] == 1.0 and r["sin_re"] == 0.0 and r["sin_im"] == 0.0
            assert r["lam1"] == a11 and r["lam2"] == a22
            assert r["perm"] == int(a11 < a22)


def test_zero_diagonal_unit_offdiagonal():
    # a11 = a22 = 0, |a21| = 1 -> lambda = (1, -1), tan = 1, sec^2 = 2
    r = O.evd2_one(False, 0.0, 0.0, 1.0, 0.0, O.EVD_TAN)
    assert (r["lam1"], r["lam2"]) == (1.0, -1.0)
    assert r["sin_re"] == 1.0 and r["cos"] == 1.0 / math.sqrt(2.0)
    r = O.evd2_one(False, 0.0, 0.0, -1.0, 0.0, O.EVD_TAN)
    assert r["sin_re"] == -1.0 and (r["lam1"], r["lam2"]) == (1.0, -1.0)


@pytest.mark.parametrize("sgn", [1.0, -1.0])
def test_evil_matrix_eq51(sgn):
    # Eq. (5.1): zeta = 0, fl(tan phi) = 1, fl(cos phi) = fl(1/fl(sqrt2)),
    # fl(e^{ia}) = 1 +- i.
    r = O.evd2_one(True, OMEGA / 8, OMEGA / 8, MU, sgn * MU, O.EVD_TAN)
    assert r["zeta"] == 0
    assert r["cos"] == 1.0 / math.sqrt(2.0) == float.fromhex("0x1.6a09e667f3bccp-1")
    assert r["sin_re"] == 1.0 and r["sin_im"] == sgn * 1.0


def test_real_equals_complex_with_zero_imag():
    # the complex algorithm on real data gives the real results
    a11, a22, a21 = synth.evd_cfg1(5000, seed=11)
    R = O.evd2_batched(a11, a22, a21)
    Z = O.evd2_batched(a11, a22, a21, np.zeros_like(a21))
    for k in ("lam1", "lam2", "cos", "sin_re", "zeta", "perm"):
        assert np.array_equal(R[k].view(np.uint8), Z[k].view(np.uint8)), k


def test_batched_equals_one_by_one_and_perm_words():
    a11, a22, re, im = synth.evd_cfg2(333, seed=12)
    B = O.evd2_batched(a11, a22, re, im)
    Bn = O.evd2_batched(a11, a22, re, im, O.EVD_NOBACKSCALE)
    for l in range(333):
        r = O.evd2_one(True, a11[l], a22[l], re[l], im[l])
        for k in ("lam1", "lam2", "cos", "sin_re", "sin_im", "zeta"):
            assert bits(float(B[k][l])) == bits(float(r[k])) if k != "zeta" else B[k][l] == r[k]
        bit = (int(B["perm"][l // 32]) >> (l % 32)) & 1
        assert bit == r["perm"] == int(Bn["lam1"][l] < Bn["lam2"][l])  # scaled values
    assert B["perm"].shape == (11,)


# ---------------------------------------------------------------- Prop 2.2 bounds
def _exact_scaled(a11, a22, re, im, z):
    """The scaled rounded matrix A' = 2^zeta A (math.ldexp is correctly rounded)."""
    return [mpmath.mpf(math.ldexp(v, z)) for v in (a11, a22, re, im)]


def _givens_batch(n, cplx, seed):
    """Eq. (2) generator: prescribed lambda, tan phi, alpha,
    assembled at 60 digits and rounded; |l1|+|l2| <= omega/8."""
    mpmath.mp.dps = 60
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        e = rng.integers(-1000, 1015, 2)
        lam = [mpmath.mpf(float(v)) for v in rng.standard_normal(2) * 2.0 ** e]
        t = mpmath.mpf(int(rng.integers(-2**62, 2**62))) / 2**62
        ca = mpmath.mpf(int(rng.integers(-2**62, 2**62))) / 2**62 if cplx else mpmath.mpf(1)
        sa = mpmath.sqrt(1 - ca * ca) * (1 if rng.random() < 0.5 else -1) if cplx else 0
        c2 = 1 / (1 + t * t)
        a11 = c2 * (lam[0] + lam[1] * t * t)
        a22 = c2 * (lam[0] * t * t + lam[1])
        off = c2 * t * (lam[0] - lam[1])
        out.append((float(a11), float(a22), float(off * ca), float(off * sa)))
    return out


@pytest.mark.parametrize("cplx", [False, True])
def test_prop22_bounds_vs_60digit_reference(cplx):
    # Eq. (prop): tan phi < 5.500001 eps (R) / 11.500004 eps (C);
    # cos phi < 8.000002 eps / 14.000006 eps; |fl(e^{ia})| within 4.000001 eps.
    # Plus eigenvalues normwise <= 8 eps (SM7.1).
    mpmath.mp.dps = 60
    tb, cb = (11.500004, 14.000006) if cplx else (5.500001, 8.000002)
    worst = dict(tan=0.0, cos=0.0, ea=0.0, lam=0.0)
    for a11, a22, re, im in _givens_batch(1500, cplx, 5 + int(cplx)):
        r = O.evd2_one(cplx, a11, a22, re, im, O.EVD_TAN | O.EVD_NOBACKSCALE)
        s11, s22, sre, sim = _exact_scaled(a11, a22, re, im, r["zeta"])
        ab = mpmath.sqrt(sre ** 2 + sim ** 2)
        a = s11 - s22
        if ab == 0 or a == 0:
            continue
        t2 = 2 * ab / abs(a)
        t = t2 / (1 + mpmath.sqrt(1 + t2 * t2))
        c = 1 / mpmath.sqrt(1 + t * t)
        if t < mpmath.mpf(2) ** -1000:  # Prop 2.2: "barring any underflow"
            continue
        worst["cos"] = max(worst["cos"], float(abs(r["cos"] / c - 1)) / EPS)
        et = mpmath.sqrt(mpmath.mpf(r["sin_re"]) ** 2 + mpmath.mpf(r["sin_im"]) ** 2)
        if not cplx:
            worst["tan"] = max(worst["tan"], float(abs(et / t - 1)) / EPS)
            # sign: e^{ia} tan phi has sign(a21) * sign(a)
            assert math.copysign(1, r["sin_re"]) == math.copysign(1, re) * (1 if a > 0 else -1)
        else:
            # |e^{ia} tan phi| / tan phi within the product of both bounds
            worst["ea"] = max(worst["ea"], float(abs(et / t - 1)) / EPS)
        lam1 = c * c * ((s22 * t + 2 * ab) * t + s11) if a > 0 else None
        # exact eigenvalues of the scaled matrix
        mid, rad = (s11 + s22) / 2, mpmath.sqrt((a / 2) ** 2 + ab ** 2)
        ex = sorted([mid + rad, mid - rad])
        got = sorted([mpmath.mpf(r["lam1"]), mpmath.mpf(r["lam2"])])
        nrm = mpmath.sqrt(ex[0] ** 2 + ex[1] ** 2)
        err = mpmath.sqrt((got[0] - ex[0]) ** 2 + (got[1] - ex[1]) ** 2) / nrm
        worst["lam"] = max(worst["lam"], float(err) / EPS)
        del lam1
    assert worst["cos"] < cb, worst
    assert worst["lam"] <= 8.0, worst
    if cplx:
        assert worst["ea"] < tb + 4.000001 + 1e-3, worst
    else:
        assert worst["tan"] < tb, worst


@pytest.mark.parametrize("cplx", [False, True])
def test_trace_and_determinant_invariants(cplx):
    # north_star: eigenvalue sum and product vs a long-double/brute-force check,
    # normwise: |l1+l2 - (a11+a22)| <= 8 eps (|l1|+|l2|); det squared scale.
    mpmath.mp.dps = 60
    for a11, a22, re, im in _givens_batch(600, cplx, 21 + int(cplx)):
        r = O.evd2_one(cplx, a11, a22, re, im, O.EVD_NOBACKSCALE)
        s11, s22, sre, sim = _exact_scaled(a11, a22, re, im, r["zeta"])
        l1, l2 = mpmath.mpf(r["lam1"]), mpmath.mpf(r["lam2"])
        scale = abs(l1) + abs(l2)
        if scale == 0:
            continue
        assert abs((l1 + l2) - (s11 + s22)) <= 8 * EPS * scale
        det = s11 * s22 - (sre ** 2 + sim ** 2)
        assert abs(l1 * l2 - det) <= 16 * EPS * scale ** 2


@pytest.mark.parametrize("cfg", [1, 2])
def test_unitarity_on_config_distributions(cfg):
    # ||U^H U - I||_F = sqrt2 |c^2 + |s|^2 - 1| <= 8 eps (north_star),
    # exact rational arithmetic; Eq. (5.1)-type inputs (scaled a21 with both
    # components subnormal, Remark 2.4) are the documented exception.
    n = 20000
    if cfg == 1:
        a11, a22, re = synth.evd_cfg1(n, seed=31)
        R = O.evd2_batched(a11, a22, re)
        im = np.zeros(n)
        si = np.zeros(n)
    else:
        a11, a22, re, im = synth.evd_cfg2(n, seed=32)
        R = O.evd2_batched(a11, a22, re, im)
        si = R["sin_im"]
    lim = Fraction(64) * Fraction(EPS) ** 2 / 2
    viol = []
    for l in range(n):
        c, sr, s_i = Fraction(R["cos"][l]), Fraction(R["sin_re"][l]), Fraction(si[l])
        d = c * c + sr * sr + s_i * s_i - 1
        if d * d > lim:
            z = int(R["zeta"][l])
            sub = all(abs(math.ldexp(v, min(z, 4096))) < 2.2250738585072014e-308
                      for v in (re[l], im[l]))
            viol.append((l, sub))
    assert all(sub for _, sub in viol), viol[:5]
    assert len(viol) <= n // 1000


def test_no_overflow_near_omega_and_subnormals():
    # Prop 2.2: scaled computations never overflow; outputs finite, no NaN.
    rng = np.random.default_rng(7)
    vals = [OMEGA, -OMEGA, OMEGA / 2, MU, -MU, 0.0, 2.0 ** -1022, 1.0]
    for _ in range(3000):
        a = [float(rng.choice(vals)) for _ in range(4)]
        r = O.evd2_one(True, *a, O.EVD_NOBACKSCALE)
        for k in ("lam1", "lam2", "cos", "sin_re", "sin_im"):
            assert math.isfinite(r[k]), (a, r)
        assert 0.0 < r["cos"] <= 1.0
    # R#7: backscaled lambda may overflow, lambda' may not
    r = O.evd2_one(True, OMEGA, OMEGA, OMEGA, OMEGA)
    assert r["lam1"] == math.inf
    r = O.evd2_one(True, OMEGA, OMEGA, OMEGA, OMEGA, O.EVD_NOBACKSCALE)
    assert math.isfinite(r["lam1"]) and r["zeta"] == -3


def test_sin_form_is_tan_form_over_sec():
    # e^{ia} sin phi = e^{ia} tan phi / sec phi; checked
    # as sin = tan * cos within 2 eps (both rounded from the same t).
    a11, a22, re, im = synth.evd_cfg2(4000, seed=41)
    S = O.evd2_batched(a11, a22, re, im)
    T = O.evd2_batched(a11, a22, re, im, O.EVD_TAN)
    for k in ("sin_re", "sin_im"):
        ok = np.abs(S[k] - T[k] * S["cos"]) <= 3 * EPS * np.abs(T[k] * S["cos"]) + 1e-300
        assert ok.all()
    assert np.array_equal(S["lam1"], T["lam1"]) and np.array_equal(S["cos"], T["cos"])
