"""Pins for the Jacobi-SVD part of the oracle (norms, dot, Gram, rotation,
strategy, step, driver).  Expected values come from the paper's worked examples,
exact rational arithmetic, 60-digit mpmath, LAPACK (numpy) and brute force --
never from the oracle itself or the CUDA path.  CPU only.
"""
import itertools
import math
from fractions import Fraction

import mpmath
import numpy as np
import pytest

import oracle as O
import synth

EPS = 2.0 ** -53
OMEGA = np.finfo(np.float64).max
R1 = O.RSpec.make(1, 1, [])
R32 = O.RSpec.make(32, 1, [16, 8, 4, 2, 1])
R256 = O.RSpec.make(256, 1, [16, 8, 4, 2, 1, 128, 64, 32])


# ---------------------------------------------------------------- (e,f) norms
def test_ef_examples_sm61():
    # 12 = (3,1.5), sqrt(12) = (1, fl(sqrt 3)); 80 = (6,1.25), sqrt = (3, fl(sqrt 1.25))
    assert O.colnorm(np.array([2.0, 2.0, 2.0]), R1) == (1.0, math.sqrt(3.0))
    assert O.colnorm(np.array([8.0, 4.0]), R1) == (3.0, math.sqrt(1.25))
    assert O.colnorm(np.array([8.0, 4.0]), R32) == (3.0, math.sqrt(1.25))
    assert O.colnorm(np.zeros(7), R32) == (-math.inf, 1.0)  # 0 = (-inf, 1)
    assert O.colnorm(np.array([0.0, 3.0 + 4.0j]), R1) == (2.0, 1.25)  # |3+4i| = 5 = 2^2 * 1.25


def test_ef_norm_of_omega_vector_is_finite():
    # x = omega * 1, m >= 2: fl(||x||) = inf but (e'', f'') finite
    for m in (2, 3, 1000):
        e, f = O.colnorm(np.full(m, OMEGA), R32)
        assert math.isfinite(e) and 1.0 <= f < 2.0
        mpmath.mp.dps = 60
        exact = mpmath.mpf(OMEGA) * mpmath.sqrt(m)
        got = mpmath.mpf(2) ** int(e) * mpmath.mpf(f)
        assert abs(got / exact - 1) < 4 * EPS


def test_ef_norm_scaling_equivariance():
    # norm(2^k x) = (e + k, f) bitwise while elements stay normal
    rng = np.random.default_rng(1)
    x = rng.standard_normal(300)
    e0, f0 = O.colnorm(x, R256)
    for k in (-900, -17, 1, 33, 900):
        assert O.colnorm(np.ldexp(x, k), R256) == (e0 + k, f0)


@pytest.mark.parametrize("cplx", [False, True])
def test_ef_norm_vs_60digit(cplx):
    # relative error <= (ceil(m/W) + lg W + 3) eps (SSQ in spec R + sqrt)
    mpmath.mp.dps = 60
    rng = np.random.default_rng(2 + cplx)
    for m, R in ((1, R1), (37, R32), (300, R32), (1000, R256), (4096, R256)):
        x = rng.standard_normal(m) * 2.0 ** rng.integers(-30, 30, m)
        if cplx:
            x = x + 1j * rng.standard_normal(m)
        e, f = O.colnorm(x, R)
        exact = mpmath.sqrt(mpmath.fsum(mpmath.mpf(abs(v.real)) ** 2 + mpmath.mpf(abs(v.imag)) ** 2
                                        for v in np.atleast_1d(x).astype(complex)))
        got = mpmath.mpf(2) ** int(e) * mpmath.mpf(f)
        bound = (math.ceil(m / R.W) * (2 if cplx else 1) + math.log2(R.W) + 3) * EPS
        assert abs(got / exact - 1) <= bound
        assert 1.0 <= f < 2.0


def test_reduction_spec_order_hand_derived():
    # R#15 pinned by hand: q = [2^53, 1, 0, 1], p = 1, norms (0, 1) (no scaling).
    #  W=1:          ((2^53 + 1) + 0) + 1  -> 2^53 (ties-to-even twice)
    #  W=2, c=1:     lane0 = 2^53 + 0, lane1 = 1 + 1 = 2 -> 2^53 + 2
    #  W=2, c=2:     lane0 = 2^53 + 1 -> 2^53, lane1 = 0 + 1 -> 2^53 + 1 -> 2^53
    q = np.array([2.0 ** 53, 1.0, 0.0, 1.0])
    p = np.ones(4)
    assert O.dot(q, 0.0, 1.0, p, 0.0, 1.0, R1)[0] == 2.0 ** 53
    assert O.dot(q, 0.0, 1.0, p, 0.0, 1.0, O.RSpec.make(2, 1, [1]))[0] == 2.0 ** 53 + 2
    assert O.dot(q, 0.0, 1.0, p, 0.0, 1.0, O.RSpec.make(2, 2, [1]))[0] == 2.0 ** 53
    # W=4, offsets [2,1]: lanes (2^53, 1, 0, 1): [1+...]: acc0 = 2^53+0, acc1 = 1+1 = 2, then 2^53 + 2
    assert O.dot(q, 0.0, 1.0, p, 0.0, 1.0, O.RSpec.make(4, 1, [2, 1]))[0] == 2.0 ** 53 + 2
    # W=4, offsets [1,2]: acc0 = 2^53+1 -> 2^53, acc2 = 0+1 = 1, then 2^53 + 1 -> 2^53
    assert O.dot(q, 0.0, 1.0, p, 0.0, 1.0, O.RSpec.make(4, 1, [1, 2]))[0] == 2.0 ** 53


# ---------------------------------------------------------------- dot, Alg 3.1
def test_dot_orthogonal_and_identical():
    x = np.zeros(64)
    y = np.zeros(64)
    x[3], y[10] = 5.0, -2.0
    ex, fx = O.colnorm(x, R32)
    ey, fy = O.colnorm(y, R32)
    assert O.dot(y, ey, fy, x, ex, fx, R32) == (0.0, 0.0)
    rng = np.random.default_rng(5)
    for cplx in (False, True):
        x = rng.standard_normal(333) + (1j * rng.standard_normal(333) if cplx else 0)
        e, f = O.colnorm(x, R32)
        zr, zi = O.dot(x, e, f, x, e, f, R32)
        assert abs(zr - 1.0) <= 16 * EPS and abs(zi) <= 16 * EPS


@pytest.mark.parametrize("cplx", [False, True])
def test_dot_vs_60digit_including_exponent_disparity(cplx):
    # huge exponent disparity e_p - e_q = 600 stays finite and accurate;
    # conjugation of q (a21' = g_q^* g_p), not of p.
    mpmath.mp.dps = 60
    rng = np.random.default_rng(6 + cplx)
    for shift in (0, 600, -600):
        m = 200
        p = rng.standard_normal(m) + (1j * rng.standard_normal(m) if cplx else 0)
        q = (0.3 * p + rng.standard_normal(m)) * 2.0 ** shift
        if cplx:
            q = q + 0.2j * p * 2.0 ** shift
        ep, fp = O.colnorm(p, R32)
        eq, fq = O.colnorm(q, R32)
        zr, zi = O.dot(q, eq, fq, p, ep, fp, R32)
        num = mpmath.fsum(mpmath.mpc(complex(a)).conjugate() * mpmath.mpc(complex(b))
                          for a, b in zip(q.astype(complex), p.astype(complex)))
        nq = mpmath.sqrt(mpmath.fsum(abs(mpmath.mpc(complex(a))) ** 2 for a in q.astype(complex)))
        npp = mpmath.sqrt(mpmath.fsum(abs(mpmath.mpc(complex(a))) ** 2 for a in p.astype(complex)))
        ex = num / (nq * npp)
        assert abs(mpmath.mpc(zr, zi) - ex) <= 64 * EPS


# ---------------------------------------------------------------- cvg, Alg 3.2
def test_convergence_threshold():
    ups = O.upsilon(4096)
    assert ups == 2.0 ** -47  # fl(2^-53 sqrt(4096))
    assert O.upsilon(64) == 2.0 ** -50
    assert O.upsilon(32768) == float.fromhex("0x1.6a09e667f3bcdp-46")
    assert O.cvg(ups, 0.0, ups)          # |z| = upsilon -> transform (">=" )
    assert not O.cvg(ups * (1 - EPS), 0.0, ups)
    assert not O.cvg(0.0, 0.0, ups)
    assert O.cvg(0.0, -ups, ups)


# ---------------------------------------------------------------- Gram, Alg 3.3
def test_gram_examples():
    # S:427-429 and P:1271-1274
    assert O.gram(0.25, 0.0, 5.0, 1.5, 5.0, 1.5) == (1.0, 1.0, 0.25, 0.0)
    a11, a22, b, bi = O.gram(0.5, -0.25, 1030.0, 1.0, 0.0, 1.0)
    assert a11 == 2.0 ** 1023 and a22 == 2.0 ** -1037  # s_A = 1023 - 1030 = -7
    assert b == 0.5 * 2.0 ** -7 and bi == -0.25 * 2.0 ** -7
    # general: a11'' a22'' = 2^{2 s_A}, ratios exact to the rounding of f1/f2
    rng = np.random.default_rng(8)
    for _ in range(500):
        e1, e2 = rng.integers(-1100, 1100, 2).astype(float)
        f1, f2 = 1 + rng.random(2)
        a11, a22, _, _ = O.gram(0.0, 0.0, e1, f1, e2, f2)
        exact = Fraction(f1) / Fraction(f2) * Fraction(2) ** int(e1 - e2)
        assert math.isfinite(a11) and math.isfinite(a22)
        # the clamp s_A <= 0 only ever scales both diagonal entries by the same 2^s_A
        if a11 > 2.0 ** -1022 and a22 > 2.0 ** -1022:
            sA = Fraction(a11) / exact
            assert abs(Fraction(a22) * exact / sA - 1) <= 4 * EPS
            k = math.log2(sA)
            assert abs(k - round(k)) < 1e-9 and round(k) <= 0
            if round(k) < 0:  # clamped: the larger entry sits at exponent 1023
                assert math.floor(math.log2(max(a11, a22))) == 1023


# ---------------------------------------------------------------- rotation, Alg 3.4
def test_rotation_lemma31_real():
    # Lemma 3.1: each output within (1 +- eps)^2 of the exact
    # transform with the same c and T; identity rotation leaves columns unchanged.
    rng = np.random.default_rng(9)
    for _ in range(200):
        p = rng.standard_normal(16) * 2.0 ** rng.integers(-300, 300)
        q = rng.standard_normal(16) * 2.0 ** rng.integers(-300, 300)
        r = O.evd2_one(False, 1.5, -0.25, rng.standard_normal(), 0.0, O.EVD_TAN)
        c, T = r["cos"], r["sin_re"]
        P2, Q2 = p.copy(), q.copy()
        M = O.rot(P2, Q2, c, T)
        for i in range(16):
            ep = (Fraction(q[i]) * Fraction(T) + Fraction(p[i])) * Fraction(c)
            eq = (-Fraction(p[i]) * Fraction(T) + Fraction(q[i])) * Fraction(c)
            for got, ex in ((P2[i], ep), (Q2[i], eq)):
                if ex != 0:
                    rel = Fraction(got) / ex
                    assert (1 - Fraction(EPS)) ** 2 <= rel <= (1 + Fraction(EPS)) ** 2
        assert M == max(np.abs(P2).max(), np.abs(Q2).max())
    p = rng.standard_normal(5)
    q = rng.standard_normal(5)
    P2, Q2 = p.copy(), q.copy()
    O.rot(P2, Q2, 1.0, 0.0)
    assert np.array_equal(P2, p) and np.array_equal(Q2, q)


def test_rotation_complex_formula_and_lemma32():
    # Eq. (transf) with e' = C + iS: x_p' = (x_p + x_q e') c, x_q' = (x_q - x_p conj(e')) c;
    # Lemma 3.2: relative error <= 5.656856 eps when |g'|/c >= |Re g_other|.
    rng = np.random.default_rng(10)
    for _ in range(200):
        p = rng.standard_normal(8) + 1j * rng.standard_normal(8)
        q = rng.standard_normal(8) + 1j * rng.standard_normal(8)
        r = O.evd2_one(True, 2.0, 1.0, *rng.standard_normal(2), O.EVD_TAN)
        c, C, S = r["cos"], r["sin_re"], r["sin_im"]
        P2, Q2 = p.copy(), q.copy()
        O.rot(P2, Q2, c, C, S)
        mpmath.mp.dps = 60
        e1 = mpmath.mpc(C, S)
        for i in range(8):
            xp, xq = mpmath.mpc(complex(p[i])), mpmath.mpc(complex(q[i]))
            ep = (xp + xq * e1) * c
            eq = (xq - xp * e1.conjugate()) * c
            if abs(ep) / c >= abs(q[i].real):
                assert abs(mpmath.mpc(complex(P2[i])) - ep) / abs(ep) <= 5.656856 * EPS
            if abs(eq) / c >= abs(p[i].real):
                assert abs(mpmath.mpc(complex(Q2[i])) - eq) / abs(eq) <= 5.656856 * EPS


def test_rotation_no_overflow_bounds():
    # Lemmas 3.1/3.2: inputs <= omega/2 (real) / omega/4 (complex) -> outputs <= omega
    rng = np.random.default_rng(11)
    for _ in range(300):
        r = O.evd2_one(True, *rng.standard_normal(4), O.EVD_TAN)
        p = (OMEGA / 4) * np.sign(rng.standard_normal(4)) * (1 + 1j)
        q = (OMEGA / 4) * np.sign(rng.standard_normal(4)) * (1 - 1j)
        P2, Q2 = p.astype(complex), q.astype(complex)
        M = O.rot(P2, Q2, r["cos"], r["sin_re"], r["sin_im"])
        assert math.isfinite(M)
        rr = O.evd2_one(False, *rng.standard_normal(3), 0.0, O.EVD_TAN)
        p = (OMEGA / 2) * np.sign(rng.standard_normal(4))
        q = (OMEGA / 2) * np.sign(rng.standard_normal(4))
        assert math.isfinite(O.rot(p.copy(), q.copy(), rr["cos"], rr["sin_re"]))


# ---------------------------------------------------------------- strategy
@pytest.mark.parametrize("n,B", [(2, 2), (4, 4), (8, 8), (8, 4), (8, 2), (12, 6), (16, 16),
                                 (16, 8), (32, 16), (64, 16), (96, 16), (128, 8), (256, 16)])
def test_strategy_exhaustive(n, B):
    # n-1 steps of n/2 disjoint pairs, every pair exactly once per sweep
    seen = set()
    for k in range(n - 1):
        pr = O.strategy_pairs(n, B, k)
        assert pr.shape == (n // 2, 2)
        assert (pr[:, 0] < pr[:, 1]).all()
        assert len(set(pr.reshape(-1).tolist())) == n
        for a, b in pr.tolist():
            assert (a, b) not in seen
            seen.add((a, b))
    assert len(seen) == n * (n - 1) // 2


def test_strategy_flat_rr_is_circle_method():
    # n = 4 by hand: round 0: (0,3), (1,2); round 1: (0,1)->pos0=0,pos3=1? see R#20
    assert O.strategy_pairs(4, 4, 0).tolist() == [[0, 3], [1, 2]]
    assert O.strategy_pairs(4, 4, 1).tolist() == [[0, 1], [2, 3]]
    assert O.strategy_pairs(4, 4, 2).tolist() == [[0, 2], [1, 3]]
    assert [O.strategy_is_checkpoint(8, 8, k) for k in range(7)] == [True] * 7
    assert [O.strategy_is_checkpoint(8, 2, k) for k in range(7)] == \
        [True, False, False, True, False, False, False]


def test_strategy_rejects_bad_args():
    for n, B in ((7, 7), (12, 4), (8, 3)):  # n odd; b = 3 odd; B does not divide n
        with pytest.raises(ValueError):
            O.strategy_pairs(n, B, 0)


# ---------------------------------------------------------------- Eqs. skn/skr
def test_Fm_exact_floors_vs_60digit():
    mpmath.mp.dps = 60
    om = mpmath.mpf(OMEGA)
    for m in list(range(1, 3000)) + [2 ** k + d for k in range(12, 40) for d in (-1, 0, 1)]:
        fr = int(mpmath.floor(mpmath.log(om / (2 * m), 2)))
        fc = int(mpmath.floor(mpmath.log(om / (4 * m * mpmath.sqrt(2)), 2)))
        assert O.Fm(False, m) == fr, m
        assert O.Fm(True, m) == fc, m
    assert O.Fm(False, 128) == 1015  # real, m = 128, M = 1 -> s0 = 1015 - 0 - 1


# ---------------------------------------------------------------- step
def test_step_skips_orthogonal_and_transforms_others():
    G = np.asfortranarray(np.diag([4.0, 1.0, 3.0, 2.0]))
    V = np.asfortranarray(np.eye(4))
    out = O.step(G, V, np.array([[0, 1], [2, 3]]), R32)
    assert out["t"] == 0 and np.array_equal(G, np.diag([4.0, 1.0, 3.0, 2.0]))
    assert out["col_e"].tolist() == [2.0, 0.0, 1.0, 1.0] and out["col_f"].tolist() == [1, 1, 1.5, 1]
    rng = np.random.default_rng(12)
    G = np.asfortranarray(rng.standard_normal((10, 4)))
    G0 = G.copy()
    V = np.asfortranarray(np.eye(4))
    out = O.step(G, V, np.array([[0, 2], [1, 3]]), R32)
    assert out["t"] == 2
    # columns of the pair are now numerically orthogonal; G V^{-1} = G0 (V orthogonal)
    for p, q in ((0, 2), (1, 3)):
        assert abs(G[:, p] @ G[:, q]) <= 64 * EPS * np.linalg.norm(G[:, p]) * np.linalg.norm(G[:, q])
    assert np.allclose(G @ V.T, G0, atol=1e-14)
    assert out["mmax"] == np.abs(G).max()


# ---------------------------------------------------------------- driver
def test_gesvj_identity_and_orthogonal_columns():
    r = O.gesvj(np.eye(6), R32)
    assert r["status"] == 0 and r["sweeps"] == 1 and r["tps"].tolist() == [0]
    assert np.array_equal(r["U"], np.eye(6)) and np.array_equal(r["V"], np.eye(6))
    assert r["sigma"].tolist() == [1.0] * 6
    # orthogonal columns with distinct norms: no transformation, sigma sorted
    G = np.diag([1.0, 4.0, 2.0, 8.0])
    r = O.gesvj(G, R32)
    assert r["tps"].tolist() == [0]
    assert r["sigma"].tolist() == [8.0, 4.0, 2.0, 1.0]
    assert r["sigma_e"].tolist() == [3.0, 2.0, 1.0, 0.0]
    assert np.array_equal(np.abs(r["V"]), np.eye(4)[:, [3, 1, 2, 0]])


def test_gesvj_errors():
    with pytest.raises(ValueError):
        O.gesvj(np.zeros((4, 4)), R32)     # ERANK
    A = np.ones((4, 4))
    A[1, 1] = np.nan
    with pytest.raises(ValueError):
        O.gesvj(A, R32)                    # ENONFINITE
    with pytest.raises(ValueError):
        O.gesvj(np.ones((3, 4)), R32)      # m < n


def _mp_svals(A):
    mpmath.mp.dps = 50
    M = mpmath.matrix(A.tolist())
    return sorted([float(v) for v in mpmath.svd_r(M, compute_uv=False)], reverse=True) \
        if not np.iscomplexobj(A) else \
        sorted([float(v) for v in mpmath.svd_c(M, compute_uv=False)], reverse=True)


@pytest.mark.parametrize("cplx", [False, True])
def test_gesvj_small_vs_mpmath(cplx):
    # relative sigma accuracy of one-sided Jacobi on well-conditioned B times
    # graded D: compare against 50-digit mpmath SVD.
    rng = np.random.default_rng(13 + cplx)
    for m, n in ((4, 2), (6, 4), (8, 6), (8, 8)):
        Bm = rng.standard_normal((m, n)) + (1j * rng.standard_normal((m, n)) if cplx else 0)
        for grade in (0, 8):
            A = Bm * (2.0 ** (-grade * np.arange(n)))
            r = O.gesvj(A, R32)
            ex = np.array(_mp_svals(A))
            assert r["status"] == 0
            rel = np.abs(r["sigma"] - ex) / ex
            assert rel.max() <= 1e-14, (m, n, grade, rel)
            U, V = r["U"], r["V"]
            assert np.linalg.norm(U.conj().T @ U - np.eye(n)) <= 64 * EPS * n
            assert np.linalg.norm(V.conj().T @ V - np.eye(n)) <= 64 * EPS * n
            res = np.linalg.norm(A - (U * r["sigma"]) @ V.conj().T) / np.linalg.norm(A)
            assert res <= 1e-14


def test_gesvj_cfg4_class_vs_lapack():
    # 64x32 complex Gaussian (kappa ~ 6): sigma vs LAPACK <= 1e-13 relative
    A = synth.svd_cfg4(3, seed=99)
    for k in range(3):
        r = O.gesvj(A[k], R32)
        s = np.linalg.svd(A[k], compute_uv=False)
        assert r["status"] == 0 and r["sweeps"] <= 15
        assert (np.abs(r["sigma"] - s) / s).max() <= 1e-13
        res = np.linalg.norm(A[k] - (r["U"] * r["sigma"]) @ r["V"].conj().T) / np.linalg.norm(A[k])
        assert res <= 1e-14


def test_gesvj_prescribed_sigma_graded():
    # A = Q1 diag(sigma) Q2^T with geometric sigma (configs[2] family, small):
    # normwise |sigma_hat - sigma| <= 10 n eps sigma_1 (R#30); residual, orthogonality.
    A, sig = synth.svd_cfg3(m=96, n=32, seed=17, kappa=1e8)
    r = O.gesvj(A, R32, max_sweeps=80)
    assert r["status"] == 0
    assert np.abs(r["sigma"] - sig).max() <= 10 * 32 * EPS * sig[0]
    n = 32
    # R#31: the north_star's n*1e-15 orthogonality is not a property of the method
    # (each of the sweeps*(n-1) rotations touching a column adds O(eps)); the pin
    # is the linear accumulation bound 4 * sweeps * n * eps.
    lim = 4 * r["sweeps"] * n * EPS
    assert np.linalg.norm(r["U"].T @ r["U"] - np.eye(n)) <= lim
    assert np.linalg.norm(r["V"].T @ r["V"] - np.eye(n)) <= lim
    res = np.linalg.norm(A - (r["U"] * r["sigma"]) @ r["V"].T) / np.linalg.norm(A)
    assert res <= 1e-13


def test_gesvj_block_strategy_converges_to_same_sigma():
    A, sig = synth.svd_cfg3(m=64, n=32, seed=18, kappa=1e4)
    a = O.gesvj(A, R32, B=32)
    b = O.gesvj(A, R32, B=4)
    assert a["status"] == b["status"] == 0
    assert np.abs(a["sigma"] - b["sigma"]).max() <= 64 * EPS * sig[0]


def test_gesvj_scale_invariance_of_bits():
    # the power-of-two prescaling makes the result exactly equivariant:
    # gesvj(2^k A) = (U, 2^k sigma, V) bitwise (s0 absorbs k)
    A = synth.svd_cfg4(1, seed=5)[0]
    r0 = O.gesvj(A, R32)
    for k in (-700, 3, 600):
        r = O.gesvj(np.ldexp(A.real, k) + 1j * np.ldexp(A.imag, k), R32)
        assert np.array_equal(r["U"], r0["U"]) and np.array_equal(r["V"], r0["V"])
        assert np.array_equal(r["sigma_f"], r0["sigma_f"])
        assert np.array_equal(r["sigma_e"], r0["sigma_e"] + k)


def test_gesvj_batched_equals_single():
    A = synth.svd_cfg4(4, seed=6)
    b = O.gesvj_batched(A, R32)
    for k in range(4):
        r = O.gesvj(A[k], R32)
        assert np.array_equal(b["U"][k], r["U"]) and np.array_equal(b["V"][k], r["V"])
        assert np.array_equal(b["sigma"][k], r["sigma"]) and b["sweeps"][k] == r["sweeps"]


# ------------------------------------------- non-convergence (Alg 4.1 line 41)
def test_gesvj_capped_zero_sweeps_returns_scaled_G():
    # "if C < S then normalize ... ; return C" -- with S = 0 no
    # sweep runs, C = S, nothing is normalised: A holds G1 = 2^s0 A exactly,
    # V = I, and (e, f) are the norms of G1's columns, in column order, NOT
    # backscaled by s.  Hand values: real m = 2: F(2) = floor(lg(omega/4)) =
    # 1021, M0 = 4 -> s0 = 1021 - 2 - 1 = 1018 (Eq. skn).  Column 1 = 2^1018
    # (3, 4): E = 1020, y = (3/4, 1), SSQ = 25/16 -> (e, f) = (1020, 5/4);
    # column 2 = 2^1018 (1, 1): E = 1018, SSQ = 2 (odd exponent) -> g = 2,
    # (e, f) = (1018, fl(sqrt 2)) (R#14).
    A = np.array([[3.0, 1.0], [4.0, 1.0]])
    r = O.gesvj(A, R32, max_sweeps=0)
    assert r["status"] == 1 and r["sweeps"] == 0 and r["scale"] == 1018
    assert np.array_equal(r["U"], np.ldexp(A, 1018))
    assert np.array_equal(r["V"], np.eye(2))
    assert r["sigma_e"].tolist() == [1020.0, 1018.0]
    assert r["sigma_f"].tolist() == [1.25, math.sqrt(2.0)]
    assert r["sigma"].tolist() == [math.ldexp(1.25, 1020), math.ldexp(math.sqrt(2.0), 1018)]


def test_gesvj_capped_one_sweep_is_unnormalized_U_sigma():
    # A = [[1, 1], [0, 1]]: one rotation diagonalises A^T A = [[1,1],[1,2]],
    # whose eigenvalues are phi^2, phi^-2 (phi the golden ratio), so after the
    # single sweep (T = 1, not converged, C = S = 1): G = U Sigma' with
    # orthogonal columns of norms 2^s phi and 2^s / phi (s = F(2) - 0 - 1 =
    # 1020), G V^T = 2^s A, and sigma' unsorted in column order.
    A = np.array([[1.0, 1.0], [0.0, 1.0]])
    phi = (1.0 + math.sqrt(5.0)) / 2.0
    r = O.gesvj(A, R32, max_sweeps=1)
    assert r["status"] == 1 and r["sweeps"] == 1 and r["tps"].tolist() == [1]
    s = r["scale"]
    assert s == 1020
    G = np.ldexp(r["U"], -s)
    V = r["V"]
    assert abs(G[:, 0] @ G[:, 1]) <= 8 * EPS
    assert np.linalg.norm(V.T @ V - np.eye(2)) <= 8 * EPS
    assert np.abs(G @ V.T - A).max() <= 8 * EPS
    sig = np.ldexp(r["sigma"], -s)
    assert sorted(sig.tolist(), reverse=True) == pytest.approx([phi, 1 / phi], rel=8 * EPS)
    for j in range(2):  # not normalised: the columns' norms are sigma'
        assert np.linalg.norm(G[:, j]) == pytest.approx(sig[j], rel=4 * EPS)
        assert r["sigma"][j] == math.ldexp(r["sigma_f"][j], int(r["sigma_e"][j]))


@pytest.mark.parametrize("cplx", [False, True])
def test_gesvj_converged_is_normalized_capped_iterate(cplx):
    # Converged in C sweeps means sweep C had T = 0 and changed nothing, so the
    # capped run with S = C - 1 ends on the same iteration matrix G: the
    # converged U must be P:1481-1485's u_j = 2^-e_j g_j / f_j of the capped
    # G (computed here with numpy's IEEE ldexp and division), sorted by
    # (e - s, f) descending (R#24), and sigma_e = e - s.
    A = synth.svd_cfg4(1, m=24, n=12, seed=31)[0]
    if not cplx:
        A = np.ascontiguousarray(A.real)
    conv = O.gesvj(A, R32, max_sweeps=60)
    C = conv["sweeps"]
    assert conv["status"] == 0 and C >= 3
    cap = O.gesvj(A, R32, max_sweeps=C - 1)
    assert cap["status"] == 1 and cap["sweeps"] == C - 1
    assert cap["scale"] == conv["scale"]
    e, f, s = cap["sigma_e"], cap["sigma_f"], cap["scale"]
    order = sorted(range(12), key=lambda j: (-(e[j] - s), -f[j], j))
    U = cap["U"]
    Uexp = np.empty_like(U)
    for r_, j in enumerate(order):
        g = U[:, j]
        if cplx:
            Uexp[:, r_] = np.ldexp(g.real, -int(e[j])) / f[j] + 1j * (np.ldexp(g.imag, -int(e[j])) / f[j])
        else:
            Uexp[:, r_] = np.ldexp(g, -int(e[j])) / f[j]
    assert np.array_equal(conv["U"], Uexp)
    assert np.array_equal(conv["V"], cap["V"][:, order])
    assert np.array_equal(conv["sigma_e"], (e - s)[order])
    assert np.array_equal(conv["sigma_f"], f[order])


# ------------------------------------------ the rescale of Eqs. skn/skr (R#40)
@pytest.mark.parametrize("a22", [0.0, 2.0 ** -30])
def test_gesvj_rescale_fires_hand_derived(a22):
    # Complex m = n = 2: F(2) = 1021 - 1 - [4 >= 8] = 1020, K = 1020 (Eq. skr
    # fires iff floor(lg M~) >= 1021).  A = [[1.5, 1.5], [0, a22]], M0 = 1.5:
    # s0 = F - 0 - 1 + adj = 1019 + adj (adj = s0_adjust).  The first rotation
    # (phi ~ pi/4) maps column 1 to ~ sqrt2 * 1.5 * 2^s0 e1 = 1.06 * 2^(s0+1).
    #  adj 0: M~1 = 1.5 * 2^1019, after the rotation 1.06 * 2^1020: never fires,
    #         s = 1019.
    #  adj 1: M~1 = 1.5 * 2^1020 (no fire at step 0), after the rotation
    #         1.06 * 2^1021 -> fires at the next check point with
    #         s_[k] = F - 1021 - 1 = -2: s = 1020 - 2 = 1018.
    #  adj 2: M~1 = 1.5 * 2^1021 -> fires at step 0, s_[0] = 1020 - 1021 - 1
    #         = -2: s = 1021 - 2 = 1019, then as adj 0.
    #  adj 3: floor(lg M~1) = 1022 -> s_[0] = -3: s = 1019.
    # Scaling by powers of two is exact here (no subnormals, no overflow), so
    # U, V, sigma (backscaled by s) are bitwise those of adj 0.
    A = np.array([[1.5, 1.5], [0.0, a22]], dtype=np.complex128)
    ref = O.gesvj(A, R32)
    assert ref["status"] == 0 and ref["scale"] == 1019
    for adj, s in ((1, 1018), (2, 1019), (3, 1019)):
        r = O.gesvj(A, R32, s0_adjust=adj)
        assert r["scale"] == s, adj
        for k in ("U", "V", "sigma", "sigma_e", "sigma_f"):
            assert np.array_equal(r[k], ref[k]), (adj, k)
        assert r["sweeps"] == ref["sweeps"] and np.array_equal(r["tps"], ref["tps"])
    with pytest.raises(ValueError):  # G1 would overflow
        O.gesvj(A, R32, s0_adjust=5)


@pytest.mark.parametrize("cplx", [False, True])
def test_gesvj_rescale_fires_mid_run_random(cplx):
    # s0_adjust = K + 1 - F(m) starts the iteration with floor(lg M~1) = K
    # (K = 1022 real, 1020 complex), so the check fires at the first check
    # point after some component reaches 2^(K+1).  Every rescale is a power
    # of two: the result equals the unadjusted run bitwise, and the final s
    # tells how far the iteration was scaled down.
    rng = np.random.default_rng(7 + cplx)
    K = 1020 if cplx else 1022
    fired = 0
    for t in range(24):
        m = int(rng.integers(2, 7))
        n = 2 * int(rng.integers(1, m // 2 + 1))
        A = rng.standard_normal((m, n)) + (1j * rng.standard_normal((m, n)) if cplx else 0)
        ref = O.gesvj(A, R32, B=n)
        adj = K + 1 - O.Fm(cplx, m)
        r = O.gesvj(A, R32, B=n, s0_adjust=adj)
        s_start = ref["scale"] + adj
        assert r["scale"] <= s_start
        fired += r["scale"] < s_start
        for k in ("U", "V", "sigma", "sigma_e", "sigma_f"):
            assert np.array_equal(r[k], ref[k]), (t, k)
        # after a rescale floor(lg M~) = F - 1, i.e. the iteration is back at
        # the paper's scale or below it
        if r["scale"] < s_start:
            assert r["scale"] <= ref["scale"]
    assert fired >= 4  # deterministic seeds: 5 (complex) of 24 fire


def test_gesvj_batched_passes_s0_adjust_and_scale():
    A = synth.svd_cfg4(3, m=8, n=4, seed=41)
    adj = 1021 - O.Fm(True, 8)
    b = O.gesvj_batched(A, R32, s0_adjust=adj)
    for k in range(3):
        r = O.gesvj(A[k], R32, s0_adjust=adj)
        assert np.array_equal(b["U"][k], r["U"]) and b["scale"][k] == r["scale"]
