"""GPU primitive tests (layer 2): the device division and scalbn
used by every kernel must equal IEEE binary64 RN arithmetic bit for bit,
including zeros, subnormals, overflow and 0/0."""
import ctypes as ct

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(mode, a, b):
    import paper_2202_08361_b200 as J
    L = J.lib()
    L.jsvd_debug_primitive.restype = ct.c_int
    L.jsvd_debug_primitive.argtypes = [ct.c_int32, ct.c_int64, ct.c_void_p, ct.c_void_p,
                                       ct.c_void_p, ct.c_void_p]
    ga, gb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    q = torch.empty_like(ga)
    assert L.jsvd_debug_primitive(mode, a.size, ct.c_void_p(ga.data_ptr()),
                                  ct.c_void_p(gb.data_ptr()), ct.c_void_p(q.data_ptr()), None) == 0
    torch.cuda.synchronize()
    return q.cpu().numpy()


def _rand_doubles(rng, n):
    """random sign/exponent/significand over the full finite range, incl. subnormals and 0"""
    e = rng.integers(0, 2047, n, dtype=np.uint64)  # biased exponent 0..2046
    m = rng.integers(0, 1 << 52, n, dtype=np.uint64)
    s = rng.integers(0, 2, n, dtype=np.uint64) << np.uint64(63)
    x = (s | (e << np.uint64(52)) | m).view(np.float64)
    x[rng.random(n) < 0.02] = 0.0
    x[rng.random(n) < 0.01] = -0.0
    return x


def _same(q, ref):
    qb, rb = q.view(np.uint64), ref.view(np.uint64)
    nan = np.isnan(ref)
    assert np.isnan(q[nan]).all()
    bad = np.nonzero((qb != rb) & ~nan)[0]
    return bad


@pytest.mark.parametrize("seed", range(4))
def test_division_full_range(seed):
    rng = np.random.default_rng(seed)
    n = 1 << 22
    a, b = _rand_doubles(rng, n), _rand_doubles(rng, n)
    with np.errstate(all="ignore"):
        ref = a / b
    for mode in (0, 1):
        bad = _same(_run(mode, a, b), ref)
        assert bad.size == 0, (mode, a[bad[:4]], b[bad[:4]])
    nz = b != 0  # the EVD's specialised divisions require a nonzero divisor
    for mode in (3, 4, 6, 10):
        bad = _same(_run(mode, a[nz], b[nz]), ref[nz])
        assert bad.size == 0, (mode, a[nz][bad[:4]], b[nz][bad[:4]])


def test_division_near_underflow_and_overflow():
    # quotients straddling the subnormal range and DBL_MAX, incl. exact ties
    rng = np.random.default_rng(7)
    n = 1 << 22
    b = (1 + rng.random(n)) * 2.0 ** rng.integers(-60, 60, n)
    target = rng.integers(-1080, -1015, n)
    q0 = (1 + rng.random(n)) * 2.0 ** 0
    a = np.ldexp(q0, target) * b
    a2 = np.ldexp(rng.integers(1, 1 << 20, n).astype(float), -1074) * 3.0  # exact multiples
    b2 = np.full(n, 3.0)
    hi = (1 + rng.random(n)) * 2.0 ** rng.integers(1015, 1023, n)
    lo = (1 + rng.random(n)) * 2.0 ** rng.integers(-12, 2, n)
    for x, y in ((a, b), (a2, b2), (hi, lo), (np.ldexp(np.ones(n), -1074), 1 + rng.random(n))):
        with np.errstate(all="ignore"):
            ref = x / y
        for mode in (0, 3, 4, 6, 10):
            bad = _same(_run(mode, x, y), ref)
            assert bad.size == 0, (mode, x[bad[:4]], y[bad[:4]])


def test_division_subnormal_ties():
    # quotients exactly at / next to a midpoint of the subnormal grid:
    # a = odd * 2^-1074 (or * 2^-1022 ... ) over b = 2, 2(1 +- ulp), 4, 6
    rng = np.random.default_rng(13)
    odd = (2 * rng.integers(0, 1 << 51, 1 << 16) + 1).astype(np.float64)
    xs, ys = [], []
    for sh in (-1074, -1073, -1060, -1023):
        for b in (2.0, 2.0 * (1 + 2.0 ** -52), 2.0 * (1 - 2.0 ** -53), 4.0, 6.0, 3.0):
            xs.append(np.ldexp(odd, sh))
            ys.append(np.full(odd.size, b))
    x, y = np.concatenate(xs), np.concatenate(ys)
    ref = x / y
    for mode in (0, 3, 4, 6, 10):
        bad = _same(_run(mode, x, y), ref)
        assert bad.size == 0, (mode, x[bad[:4]], y[bad[:4]])


def test_division_structured_significands():
    # all-ones / all-zeros / single-bit significands of both operands, every
    # combination, at exponent offsets around the normal/subnormal boundary
    sig = [1.0, 2.0 - 2.0 ** -52, 1.5, 1.0 + 2.0 ** -52, 1.5 - 2.0 ** -52, 1.25, 1.75 + 2.0 ** -52,
           1.0 + 2.0 ** -26, 2.0 - 2.0 ** -26, 1.3333333333333333, 1.6666666666666667]
    rng = np.random.default_rng(3)
    sig += list(1 + rng.random(40))
    ea = [-1074, -1060, -1030, -1023, -1022, -1000, -500, -3, 0, 1, 500, 1000, 1021, 1023]
    A, B = [], []
    for a in sig:
        for b in sig:
            for x in ea:
                for y in ea:
                    A.append(np.ldexp(a, x))
                    B.append(np.ldexp(b, y))
    a, b = np.array(A), np.array(B)
    with np.errstate(all="ignore"):
        ref = a / b
    for mode in (0, 1, 3, 4, 6, 10):
        bad = _same(_run(mode, a, b), ref)
        assert bad.size == 0, (mode, a[bad[:4]], b[bad[:4]])


def test_division_double_rounding_midpoints():
    # mode 10 rounds a subnormal result from the correctly rounded quotient Q
    # of the normalised operands: wrong exactly when Q 2^k is a midpoint of the
    # 2^-1074 grid while Q is inexact.  Build such cases: M a 53-bit
    # significand whose low s bits are 10...0, Q = M 2^-52, b random, a =
    # RN(Q b) 2^(eb - 1022 - s) over b 2^eb (so the s low bits of Q fall below
    # the subnormal grid); keep the pairs where RN(a/b) at full precision is Q and
    # the quotient is inexact (checked with exact rationals).  Both signs,
    # divisors at several exponents.
    from fractions import Fraction
    rng = np.random.default_rng(17)
    A, B = [], []
    while len(A) < 4000:
        s = int(rng.integers(1, 53))
        M = (int(rng.integers(1 << 52, 1 << 53)) >> s << s) | (1 << (s - 1))
        Q = M * 2.0 ** -52
        b = float(1 + rng.random())
        a = Q * b
        if a / b != Q or Fraction(a) / Fraction(b) == Fraction(Q):
            continue
        eb = int(rng.integers(s, 1000))
        E = eb - 1022 - s
        sg = -1.0 if rng.random() < 0.5 else 1.0
        sb = -1.0 if rng.random() < 0.3 else 1.0
        A.append(sg * np.ldexp(a, E))
        B.append(sb * np.ldexp(b, eb))
    a, b = np.array(A), np.array(B)
    ref = a / b
    assert (np.abs(ref) < 2.0 ** -1022).all()
    for mode in (0, 3, 10):
        bad = _same(_run(mode, a, b), ref)
        assert bad.size == 0, (mode, a[bad[:4]], b[bad[:4]])


def test_hypot_exact_shortcut_matches_oracle():
    import oracle as O
    rng = np.random.default_rng(21)
    n = 1 << 16
    x = np.abs(_rand_doubles(rng, n))
    y = x * 2.0 ** rng.integers(-60, 60, n) * (1 + rng.random(n))
    y[::7] = 0.0
    g = _run(5, x, y)
    ref = np.array([O.hypot(a, b) for a, b in zip(x, y)])
    bad = _same(g, ref)
    assert bad.size == 0, (x[bad[:4]], y[bad[:4]])


def test_scalbn_full_range():
    rng = np.random.default_rng(11)
    n = 1 << 22
    a = _rand_doubles(rng, n)
    k = rng.integers(-2200, 2200, n)
    ref = np.ldexp(a, k)
    bad = _same(_run(2, a, k.astype(np.float64)), ref)
    assert bad.size == 0, (a[bad[:4]], k[bad[:4]])


def test_sqrt_plain_in_range():
    # the EVD's and the norms' sqrt: arguments in [1, 4) and up to DBL_MAX
    rng = np.random.default_rng(17)
    n = 1 << 22
    xs = [1 + 3 * rng.random(n), np.ldexp(1 + rng.random(n), rng.integers(-969, 1024, n)),
          np.nextafter(np.ldexp(np.ones(n), rng.integers(-969, 1023, n)), np.inf),
          np.array([1.0, 2.0, 4.0 - 2.0 ** -50, 1 + 2.0 ** -52, np.finfo(float).max, 2.0 ** -969])]
    for x in xs:
        bad = _same(_run(7, x, x), np.sqrt(x))
        assert bad.size == 0, x[bad[:4]]


def test_div_plain_in_range():
    # the plain division on operands inside its proven range (jsvd.h)
    rng = np.random.default_rng(19)
    n = 1 << 22
    b = np.ldexp(1 + rng.random(n), rng.integers(-1000, 1000, n))
    q = np.ldexp(1 + rng.random(n), rng.integers(-999, 999, n))
    a = q * b
    ok = (np.abs(a) >= 2.0 ** -968) & np.isfinite(a) & (np.abs(a / b) >= 2.0 ** -1000) \
        & (np.abs(a / b) <= 2.0 ** 1000)
    a, b = a[ok], b[ok]
    a[::3] = -a[::3]
    b[::5] = -b[::5]
    bad = _same(_run(8, a, b), a / b)
    assert bad.size == 0, (a[bad[:4]], b[bad[:4]])
    # structured significands (ties of the Markstein step), unit exponents
    sig = np.array([1.0, 2.0 - 2.0 ** -52, 1.5, 1.0 + 2.0 ** -52, 1.5 - 2.0 ** -52, 1.25,
                    1.75 + 2.0 ** -52, 1.0 + 2.0 ** -26, 2.0 - 2.0 ** -26, 1.3333333333333333])
    A, B = np.meshgrid(np.concatenate([sig, 1 + rng.random(300)]),
                       np.concatenate([sig, 1 + rng.random(300)]))
    for ea, eb in ((0, 0), (-968, 0), (500, -400), (0, 999), (-500, -999)):
        x, y = np.ldexp(A.ravel(), ea), np.ldexp(B.ravel(), eb)
        bad = _same(_run(8, x, y), x / y)
        assert bad.size == 0, (ea, eb, x[bad[:4]], y[bad[:4]])


def test_divide_small_full_dividend_range():
    # a / d, d in [1, 2], a anywhere (subnormal quotients, exact ties on the
    # subnormal grid, signed zeros): the EVD's e^{ia} sin(phi) = e^{ia} tan / sec
    rng = np.random.default_rng(23)
    n = 1 << 22
    d = np.concatenate([1 + rng.random(n), np.array([1.0, 2.0, np.sqrt(2.0), 2.0 - 2.0 ** -52])])
    a = _rand_doubles(rng, d.size)
    a[::5] = np.ldexp(1 + rng.random(a[::5].size), rng.integers(-1080, -1000, a[::5].size))
    a[::7] *= -1
    a[3] = -0.0
    bad = _same(_run(9, a, d), a / d)
    assert bad.size == 0, (a[bad[:4]], d[bad[:4]])
    # exact ties of the final rounding (a = odd 2^-1074, d = 2: a/d is a midpoint
    # of the subnormal grid; exact ties need d a power of two) and near ties
    odd = (2 * rng.integers(0, 1 << 51, 1 << 16) + 1).astype(np.float64)
    x = np.ldexp(odd, -1074)
    for dv in (2.0, 2.0 - 2.0 ** -52, 1.0 + 2.0 ** -52, 1.0, 1.5, 1.0 + 2.0 ** -26):
        dd = np.full(x.size, dv)
        for y in (x, -x):
            bad = _same(_run(9, y, dd), y / dd)
            assert bad.size == 0, (dv, y[bad[:4]])


def test_copy16_diagnostic():
    # jsvd_copy16 (the bench's streaming-copy context line) copies exactly
    import paper_2202_08361_b200 as J
    src = torch.randn(1000002, dtype=torch.float64, device="cuda")
    dst = torch.empty_like(src)
    J.copy16(src, dst)
    torch.cuda.synchronize()
    assert torch.equal(src, dst)
    with pytest.raises(ValueError):
        J.copy16(src[:3], dst[:3])
