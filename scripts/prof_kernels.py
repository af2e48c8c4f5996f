"""Small driver for ncu captures of the SVD kernels (one launch each)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2202_08361_b200 as J
import synth

what = sys.argv[1]
if what == 'batched':
    b = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
    A = synth.svd_cfg4(b)
    g = torch.from_numpy(np.ascontiguousarray(np.transpose(A, (0, 2, 1)))).cuda()
    for _ in range(2):
        x = g.clone()
        J.gesvj_batched(x.transpose(1, 2))
    torch.cuda.synchronize()
elif what == 'step':
    A, _ = synth.svd_cfg3()
    m, n = A.shape
    s0 = (1022 - int(np.floor(np.log2(m)))) - int(np.floor(np.log2(np.abs(A).max()))) - 1
    G = torch.from_numpy(np.ascontiguousarray(np.ldexp(A, s0).T)).cuda().T
    V = torch.eye(n, dtype=torch.float64, device='cuda').T
    for k in range(8):
        J.sweep_step(G, V, J.strategy_pairs(n, n, k))
    torch.cuda.synchronize()
print('ok')
