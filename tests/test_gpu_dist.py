"""The column-block-sharded SVD with the library's kernels on one GPU: P = 1,
2, 4, 8 virtual ranks (LocalRanks: device copies for the block exchange; the
ranks run one after another, no kernel waits on another).  Results must be
bitwise identical for every P, to jsvd_gesvj(nblocks=16) and to the oracle."""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu


def _bits(a):
    a = np.ascontiguousarray(a)
    return (a.view(np.float64) if np.iscomplexobj(a) else a).view(np.uint64)


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("m,n", [(64, 32), (300, 64), (2049, 96)])
def test_dist_virtual_ranks_bitwise(cplx, m, n):
    import paper_2202_08361_b200 as J
    from paper_2202_08361_b200.dist import (BlockSchedule, CudaCompute, LocalRanks,
                                            gather_columns, gesvj_dist, scatter_columns)
    rng = np.random.default_rng(m + n + cplx)
    A = rng.standard_normal((m, n)) * 2.0 ** rng.integers(-20, 20, n)
    if cplx:
        A = A + 1j * rng.standard_normal((m, n))
    R = O.RSpec.make(*J.step_rspec(cplx, m))
    ref = O.gesvj(A, R, B=16, max_sweeps=30)
    g = torch.from_numpy(np.ascontiguousarray(A.T)).cuda().T
    lib = J.gesvj(g, nblocks=16, max_sweeps=30)
    assert np.array_equal(_bits(lib["U"].T.contiguous().cpu().numpy().T), _bits(ref["U"]))
    dt = torch.complex128 if cplx else torch.float64
    for P in (1, 2, 4, 8):
        S = BlockSchedule(n, 16, P)
        Gts = [torch.from_numpy(np.ascontiguousarray(A[:, scatter_columns(None, S, r)].T))
               .to(dt).cuda() for r in range(P)]
        res = gesvj_dist(Gts, S, LocalRanks(P), CudaCompute(), cplx=cplx)
        assert res["sweeps"] == ref["sweeps"] and list(res["tps"]) == list(ref["tps"])
        U = np.array(gather_columns([G.cpu().numpy() for G in res["Gts"]], S)).T
        V = np.array(gather_columns([V.cpu().numpy() for V in res["Vts"]], S)).T
        perm = res["perm"]
        assert np.array_equal(_bits(U[:, perm]), _bits(ref["U"])), P
        assert np.array_equal(_bits(V[:, perm]), _bits(ref["V"])), P
        assert np.array_equal(_bits(res["sigma"]), _bits(ref["sigma"]))
        assert np.array_equal(_bits(res["sigma_e"]), _bits(ref["sigma_e"]))
