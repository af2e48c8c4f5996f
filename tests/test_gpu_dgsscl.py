"""GPU parity of jsvd_dgsscl (NEXT-4, the real Gram-Schmidt orthogonalization
of Alg SM8.1 / Eq. (DGS)) against the oracle, BITWISE, on pair batches with
norms from the library's own jsvd_colnorms and scaled dots from the oracle:
ragged m, wide exponent ranges (subnormal results of scalef included), zero
columns, and a large pair batch."""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def J():
    import paper_2202_08361_b200 as J
    assert torch.cuda.is_available()
    return J


def _run(J, A, pairs, a21, ld_pad=0):
    m, n = A.shape
    buf = np.zeros((n, m + ld_pad))
    buf[:, :m] = A.T
    g = torch.from_numpy(buf).cuda().T[:m, :]
    ce, cf = J.colnorms(g)
    J.dgsscl(g, torch.from_numpy(pairs.astype(np.int32)).cuda(), ce, cf,
             torch.from_numpy(a21).cuda())
    torch.cuda.synchronize()
    got = g.T.contiguous().cpu().numpy().T
    ce, cf = ce.cpu().numpy(), cf.cpu().numpy()
    ref = np.array(A, copy=True)
    for l, (p, q) in enumerate(pairs):
        ref[:, q] = O.dgsscl(A[:, p], A[:, q], ce[p], cf[p], ce[q], cf[q], a21[l])
    assert np.array_equal(np.ascontiguousarray(got).view(np.uint64),
                          np.ascontiguousarray(ref).view(np.uint64))


@pytest.mark.parametrize("m", [1, 7, 255, 1024, 1025, 5000])
def test_dgsscl_bitwise(J, m):
    rng = np.random.default_rng(m)
    n = 16
    A = rng.standard_normal((m, n)) * 2.0 ** rng.integers(-60, 60, (m, n))
    A[:, :8] *= 2.0 ** 900   # g_p huge ...
    A[:, 8:] *= 2.0 ** -900  # ... g_q tiny: tan(phi) would underflow
    pairs = np.stack([np.arange(8), np.arange(8, 16)], axis=1)
    a21 = rng.uniform(-1, 1, 8)
    _run(J, A, pairs, a21, ld_pad=3)


def test_dgsscl_zero_column_and_subnormal_results(J):
    rng = np.random.default_rng(4)
    m, n = 600, 6
    A = rng.standard_normal((m, n))
    A[:, 1] = 0.0  # zero g_q: left as it is
    A[:, 3] *= 2.0 ** -1000
    A[:, 5] *= 2.0 ** 1000
    pairs = np.array([[0, 1], [2, 3], [4, 5]])
    _run(J, A, pairs, np.array([0.5, -0.999, 1e-300]))


def test_dgsscl_many_pairs(J):
    rng = np.random.default_rng(9)
    m, n = 2048, 512
    A = rng.standard_normal((m, n))
    pairs = rng.permutation(n).reshape(-1, 2)
    _run(J, A, pairs, rng.uniform(-1, 1, n // 2))
