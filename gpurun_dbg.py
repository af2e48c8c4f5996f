import numpy as np, torch, sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle as O, paper_2202_08361_b200 as J
from test_gpu_dist import _case, _rspec
m, n = 96, 64
for cplx in (False,):
    A = _case(cplx, m, n, seed=3)
    K = 1022
    adj = K + 1 - O.Fm(cplx, m)
    ref = O.gesvj(A, _rspec(cplx, m), B=16, max_sweeps=30, s0_adjust=adj)
    for B in (16, 64):
        refB = O.gesvj(A, _rspec(cplx, m), B=B, max_sweeps=30, s0_adjust=adj)
        g = torch.from_numpy(np.ascontiguousarray(A.T)).cuda().T
        out = J.gesvj(g, nblocks=B, max_sweeps=30, s0_adjust=adj)
        print("B", B, "gpu tps", out["tps"][:6], "scale", out["scale"], "sweeps", out["sweeps"])
        print("B", B, "orc tps", list(refB["tps"][:6]), "scale", refB["scale"], "sweeps", refB["sweeps"])
    # no adjust
    for B in (16,):
        refB = O.gesvj(A, _rspec(cplx, m), B=B, max_sweeps=30)
        g = torch.from_numpy(np.ascontiguousarray(A.T)).cuda().T
        out = J.gesvj(g, nblocks=B, max_sweeps=30)
        print("noadj B", B, out["tps"][:6], list(refB["tps"][:6]))
