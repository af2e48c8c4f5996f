import numpy as np, torch, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle as O, paper_2202_08361_b200 as J
from test_gpu_svd import _scaled_input, rspec, colmajor_gpu, to_np
for cplx in (False, True):
    m = 64; n = 12
    rng = np.random.default_rng(m + 7 * cplx)
    A = _scaled_input(rng, m, n, cplx)
    V = np.asfortranarray(np.eye(n, dtype=A.dtype) + 0.0)
    R = rspec(J, cplx, m)
    G_ref, V_ref = A.copy(order="F"), V.copy(order="F")
    g, v = colmajor_gpu(A), colmajor_gpu(V)
    pairs = O.strategy_pairs(n, n, 0)
    ref = O.step(G_ref, V_ref, pairs, R)
    out = J.sweep_step(g, v, torch.from_numpy(pairs.astype(np.int32)).cuda())
    torch.cuda.synchronize()
    ce, cf = out["col_e"].cpu().numpy(), out["col_f"].cpu().numpy()
    print("cplx", cplx, "pairs", pairs.tolist())
    for j in range(n):
        print(j, ce[j], ref["col_e"][j], cf[j], ref["col_f"][j], "OK" if (ce[j] == ref["col_e"][j] and cf[j] == ref["col_f"][j]) else "DIFF")
