"""Pins of the oracle's one-pass (e, f) Frobenius norm (NEXT-3, Alg SM6.3,
P:3040-3404; readings R#35-R#38) against things other than itself: the
paper's worked examples, exact sums of squares (Python
fractions), scale equivariance, the complex/real layout identity, the
single-element case, and a relative error bound against exact arithmetic."""
from fractions import Fraction

import numpy as np
import pytest

import oracle as O

OMEGA = float(np.finfo(np.float64).max)
MU = float(np.finfo(np.float64).smallest_subnormal)


def _ef_exact(S):
    """(e, f) of a positive Fraction S: S = 2^e f, f in [1, 2)."""
    e = S.numerator.bit_length() - S.denominator.bit_length()
    if Fraction(2) ** e > S:
        e -= 1
    if Fraction(2) ** (e + 1) <= S:
        e += 1
    return e, S / Fraction(2) ** e


def _ssq_exact(x):
    if np.iscomplexobj(x):
        return sum(Fraction(float(v.real)) ** 2 + Fraction(float(v.imag)) ** 2 for v in x)
    return sum(Fraction(float(v)) ** 2 for v in x)


@pytest.mark.parametrize("s", [1, 2, 8, 32])
def test_paper_examples_12_and_80(s):
    # 12 = (3, 1.5), sqrt 12 = (1, fl(sqrt 3)); 80 = (6, 1.25), sqrt 80 = (3, fl(sqrt 1.25))
    e, f, e2, f2 = O.norm_ef(np.array([2.0, 2.0, 2.0]), s=s)
    assert (e2, f2) == (3.0, 1.5) and (e, f) == (1.0, float(np.sqrt(3.0)))
    e, f, e2, f2 = O.norm_ef(np.array([8.0, 4.0]), s=s)
    assert (e2, f2) == (6.0, 1.25) and (e, f) == (3.0, float(np.sqrt(1.25)))


@pytest.mark.parametrize("m", [2, 4, 16, 1000])
def test_omega_vector_stays_finite(m):
    # x = omega 1 has ||x|| = omega sqrt(m) > omega, yet (e'', f'') is finite
    e, f, e2, f2 = O.norm_ef(np.full(m, OMEGA), s=8)
    assert np.isfinite(e) and np.isfinite(f) and 1.0 <= f < 2.0
    exact = Fraction(OMEGA) ** 2 * m
    ee, ff = _ef_exact(exact)
    assert e2 == ee
    assert abs(Fraction(f2) - ff) <= ff * Fraction(m + 8, 2 ** 52)


def test_zero_and_padding():
    assert O.norm_ef(np.zeros(7), s=4) == (-np.inf, 1.0, -np.inf, 1.0)   # 0 = (-inf, 1)
    assert O.norm_ef(np.zeros(0), s=4) == (-np.inf, 1.0, -np.inf, 1.0)
    x = np.array([3.0, -1.5, 0.25, 7.0, 1e-300])
    # explicit zero padding (Eq. pad0) leaves the result unchanged
    assert O.norm_ef(x, s=8) == O.norm_ef(np.concatenate([x, np.zeros(11)]), s=8)


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("scale", [0, -1070, -600, 400, 960])
def test_exact_sums_of_squares(cplx, scale):
    # integers times a common power of two: every partial sum is exact, so the
    # result is the exact (e, f) of the sum of squares -- even in the subnormal range
    rng = np.random.default_rng(abs(scale) + cplx)
    m = 300
    x = rng.integers(-1000, 1001, m).astype(np.float64)
    if cplx:
        x = x + 1j * rng.integers(-1000, 1001, m)
    x = x * 2.0 ** max(scale, -1000) * 2.0 ** min(scale + 1000, 0)  # exact; -1070: subnormal
    for s in (1, 8, 32):
        e, f, e2, f2 = O.norm_ef(x, s=s)
        ee, ff = _ef_exact(_ssq_exact(x))
        assert (e2, Fraction(f2)) == (ee, ff), (s, e2, f2, ee, float(ff))


@pytest.mark.parametrize("cplx", [False, True])
def test_scale_equivariance_bitwise(cplx):
    # the method touches only exponent differences and F(x): x -> 2^k x shifts e
    # by 2k and leaves f unchanged, bit for bit, subnormal inputs included
    rng = np.random.default_rng(11)
    m = 257
    x = rng.standard_normal(m) * 2.0 ** rng.integers(-30, 30, m)
    if cplx:
        x = x + 1j * rng.standard_normal(m) * 2.0 ** rng.integers(-30, 30, m)
    for s in (4, 32):
        for red in (0, 1):
            e0, f0, e20, f20 = O.norm_ef(x, s=s, reduction=red)
            for k in (-980, -700, 500, 950):  # every y stays normal
                y = x * 2.0 ** k
                if cplx:
                    assert np.array_equal(y.real / 2.0 ** k, x.real)  # scaling was exact
                else:
                    assert np.array_equal(y / 2.0 ** k, x)
                e, f, e2, f2 = O.norm_ef(y, s=s, reduction=red)
                assert (e2, f2) == (e20 + 2 * k, f20)
                assert f == f0 and e == e0 + k


def test_scale_equivariance_into_subnormals():
    # entries that become subnormal: getexp/getmant are exact there (R#35)
    x = np.array([1.0, 3.0, 0.5, 0.75, 1.25, 7.0, 2.0 ** -10, 1.5])
    base = O.norm_ef(x, s=4)
    y = x * 2.0 ** -1060
    assert np.count_nonzero(np.abs(y) < np.finfo(float).tiny) == len(x)
    assert np.array_equal(y * 2.0 ** 1000 * 2.0 ** 60, x)  # exact (few significant bits)
    e, f, e2, f2 = O.norm_ef(y, s=4)
    assert (e2, f2) == (base[2] - 2120, base[3])


def test_single_element_is_its_own_norm():
    rng = np.random.default_rng(3)
    for v in list(rng.standard_normal(50) * 2.0 ** rng.integers(-1070, 1020, 50)) + [MU, OMEGA, -1.0]:
        e, f, _, _ = O.norm_ef(np.array([v]), s=8)
        m, ex = np.frexp(abs(v))
        assert (e, f) == (float(ex - 1), float(m * 2))  # sqrt(RN(F^2)) = F in radix 2


@pytest.mark.parametrize("s", [4, 32])
def test_complex_is_the_interleaved_real_layout(s):
    # R#36: each iteration takes the real parts of s elements, then their imaginary parts
    rng = np.random.default_rng(9)
    m = 5 * s
    z = rng.standard_normal(m) * 2.0 ** rng.integers(-200, 200, m) + \
        1j * rng.standard_normal(m) * 2.0 ** rng.integers(-200, 200, m)
    y = np.empty(2 * m)
    for it in range(m // s):
        y[2 * it * s:(2 * it + 1) * s] = z[it * s:(it + 1) * s].real
        y[(2 * it + 1) * s:(2 * it + 2) * s] = z[it * s:(it + 1) * s].imag
    for red in (0, 1):
        assert O.norm_ef(z, s=s, reduction=red) == O.norm_ef(y, s=s, reduction=red)


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("red", [0, 1])
def test_relative_error_bound(cplx, red):
    # wide exponent range (no overflow or underflow anywhere in (e, f) form)
    rng = np.random.default_rng(21 + cplx + 2 * red)
    m = 400
    x = rng.standard_normal(m) * 2.0 ** rng.integers(-500, 500, m)
    if cplx:
        x = x + 1j * rng.standard_normal(m) * 2.0 ** rng.integers(-500, 500, m)
    S = _ssq_exact(x)
    for s in (1, 8, 32):
        e, f, e2, f2 = O.norm_ef(x, s=s, reduction=red)
        got = Fraction(f2) * Fraction(2) ** int(e2)
        assert abs(got - S) <= S * Fraction(2 * m + 2 * s, 2 ** 53)
        # the root: one more rounding (sqrt) and the exact halving of e
        r2 = Fraction(f) ** 2 * Fraction(2) ** (2 * int(e))
        assert abs(r2 - S) <= S * Fraction(2 * m + 2 * s + 4, 2 ** 53)


def test_sorting_makes_reduction_order_free():
    # the same multiset of lane sums in any lane order gives the same result:
    # permuting whole s-blocks' lanes consistently permutes the final partial sums
    rng = np.random.default_rng(17)
    s, it = 8, 6
    x = rng.standard_normal(s * it) * 2.0 ** rng.integers(-40, 40, s * it)
    perm = rng.permutation(s)
    y = x.reshape(it, s)[:, perm].reshape(-1)
    for red in (0, 1):
        assert O.norm_ef(x, s=s, reduction=red) == O.norm_ef(y, s=s, reduction=red)


def test_rejects_non_power_of_two_lanes():
    with pytest.raises(ValueError):
        O.norm_ef(np.ones(4), s=3)
