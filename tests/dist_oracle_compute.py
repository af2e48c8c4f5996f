"""TEST INFRASTRUCTURE: a compute backend for paper_2202_08361_b200.dist that
runs each block operation with the oracle on torch CPU tensors, so the
distributed schedule (block ordering, exchanges, collectives, check points,
finalize) can be exercised with gloo on CPU.  Never used by the product path."""
import math

import numpy as np
import torch

import oracle as O


def _f64(x):
    """float64 view of a real or complex numpy array."""
    return x.view(np.float64) if np.iscomplexobj(x) else x


class OracleCompute:
    def __init__(self, R):
        self.R = R

    def scalar(self, v, like):
        return torch.tensor([float(v)], dtype=torch.float64)

    def counter(self, like):
        return torch.zeros(1, dtype=torch.int64)

    def maxnorm(self, Gt, out):
        a = np.abs(_f64(Gt.numpy()))
        v = math.inf if np.isnan(a).any() else (float(a.max()) if a.size else 0.0)
        out.fill_(max(out.item(), v))

    def scale(self, Gt, s):
        x = _f64(Gt.numpy())
        x[...] = np.ldexp(x, s)  # correctly rounded scalbn

    def step(self, Gt, Vt, pairs, key, t_dev, mt_dev, ce, cf):
        G, V = Gt.numpy().T, Vt.numpy().T  # column-major views, modified in place
        out = O.step(G, V, pairs, self.R)
        t_dev += out["t"]
        mt_dev.fill_(max(mt_dev.item(), out["mmax"]))
        used = np.unique(pairs.reshape(-1))
        ce.numpy()[used] = out["col_e"][used]
        cf.numpy()[used] = out["col_f"][used]

    def colnorms(self, Gt):
        G = Gt.numpy()
        ef = [O.colnorm(np.ascontiguousarray(G[j]), self.R) for j in range(G.shape[0])]
        return (torch.tensor([e for e, _ in ef], dtype=torch.float64),
                torch.tensor([f for _, f in ef], dtype=torch.float64))

    def normalize(self, Gt, ce, cf):
        G = Gt.numpy()
        for j in range(G.shape[0]):
            e = ce[j].item()
            if not math.isinf(e):
                x = _f64(G[j])
                x[...] = np.ldexp(x, -int(e)) / cf[j].item()
