"""GPU parity of jsvd_norm_ef (NEXT-3, the one-pass (e, f) norm of Alg SM6.3)
against the oracle with s = 32 lanes and the pairwise reduction, BITWISE on
(e'', f'') and on the squared norm's (e, f).  Columns span the whole exponent
range: subnormal, huge (omega), zero, single-element and ragged lengths."""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu

OMEGA = float(np.finfo(np.float64).max)
MU = float(np.finfo(np.float64).smallest_subnormal)


@pytest.fixture(scope="module")
def J():
    import paper_2202_08361_b200 as J
    assert torch.cuda.is_available()
    return J


def _cols(rng, m, n, cplx, lo=-1070, hi=1020):
    def part():
        return rng.standard_normal((m, n)) * 2.0 ** rng.integers(lo, hi, (m, n))
    A = part() + 1j * part() if cplx else part()
    A[rng.random((m, n)) < 0.05] = 0.0
    return A


def _gpu_colmajor(A, ld_pad=0):
    m, n = A.shape
    buf = np.zeros((n, m + ld_pad), dtype=A.dtype)
    buf[:, :m] = A.T
    t = torch.from_numpy(buf).cuda()
    return t.T[:m, :]  # (m, n) view with ld = m + ld_pad


def _check(J, A, ld_pad=0):
    g = _gpu_colmajor(A, ld_pad)
    n = A.shape[1]
    e2 = torch.empty(n, dtype=torch.float64, device="cuda")
    f2 = torch.empty(n, dtype=torch.float64, device="cuda")
    ce, cf = J.norm_ef(g, col_e2=e2, col_f2=f2)
    torch.cuda.synchronize()
    ce, cf, e2, f2 = (t.cpu().numpy() for t in (ce, cf, e2, f2))
    for j in range(n):
        ref = O.norm_ef(A[:, j], s=32, reduction=0)
        got = (ce[j], cf[j], e2[j], f2[j])
        assert np.array_equal(np.array(got).view(np.uint64), np.array(ref).view(np.uint64)), \
            (j, got, ref)


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("m", [1, 5, 31, 32, 33, 127, 128, 129, 1000, 4099])
def test_norm_ef_bitwise_ragged(J, cplx, m):
    rng = np.random.default_rng(m + 7 * cplx)
    _check(J, _cols(rng, m, 19, cplx))


@pytest.mark.parametrize("cplx", [False, True])
def test_norm_ef_special_columns(J, cplx):
    m = 300
    rng = np.random.default_rng(44)
    cols = [np.zeros(m), np.full(m, OMEGA), np.full(m, MU), np.full(m, -OMEGA),
            np.where(np.arange(m) == 77, 3.0, 0.0),                       # single element
            rng.standard_normal(m) * 2.0 ** -1060,                        # subnormal
            np.concatenate([np.full(m // 2, OMEGA), np.full(m - m // 2, MU)]),  # both ends
            rng.standard_normal(m) * 2.0 ** rng.integers(-1074, 1023, m)]
    A = np.stack(cols, axis=1)
    if cplx:
        A = A + 1j * np.stack(cols[::-1], axis=1)
    _check(J, A)


@pytest.mark.parametrize("cplx", [False, True])
def test_norm_ef_leading_dimension_and_narrow_range(J, cplx):
    rng = np.random.default_rng(3)
    _check(J, _cols(rng, 777, 9, cplx, -5, 5), ld_pad=13)


@pytest.mark.parametrize("cplx", [False, True])
def test_norm_ef_large_sampled(J, cplx):
    # many columns at a bench-like column length: every column of a 32768 x 64
    # matrix against the oracle
    rng = np.random.default_rng(8)
    A = _cols(rng, 32768, 64 if cplx else 96, cplx, -200, 200)
    _check(J, A)


def test_norm_ef_agrees_with_two_level_norm(J):
    # the same norms as jsvd_colnorms (R#14) up to a few ulps (different summation)
    rng = np.random.default_rng(12)
    A = rng.standard_normal((4096, 40)) * 2.0 ** rng.integers(-20, 20, (1, 40))
    g = _gpu_colmajor(A)
    ce, cf = J.norm_ef(g)
    ce2, cf2 = J.colnorms(g)
    a = np.ldexp(cf.cpu().numpy(), ce.cpu().numpy().astype(int))
    b = np.ldexp(cf2.cpu().numpy(), ce2.cpu().numpy().astype(int))
    assert np.max(np.abs(a - b) / b) < 64 * 2.0 ** -53


def test_norm_ef_empty_and_errors(J):
    g = torch.zeros((0, 4), dtype=torch.float64, device="cuda")
    ce, cf = J.norm_ef(g)
    torch.cuda.synchronize()
    assert np.all(np.isneginf(ce.cpu().numpy())) and np.all(cf.cpu().numpy() == 1.0)
    import ctypes as ct
    L = J.lib()
    assert L.jsvd_norm_ef(1, 4, 4, None, 2, None, None, None, None, None) == -1  # ld < m
