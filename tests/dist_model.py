"""TEST INFRASTRUCTURE: a CPU model of the sharded jsvd_gesvj driver
(gesvj.cu with a jsvd_dist) -- the same slot layout, the library's own local
pair schedule (jsvd_dist_local_pairs, a host-only C function), the block moves
after every phase-II round (position k -> k-1, 1 -> B-1, 0 stays: restated
here), the global M-tilde at the check points and the global sort -- with the
oracle as compute and a paper_2202_08361_b200.dist transport (ThreadGroup or
GlooTransport) for the collectives.  It lets the CPU suite check, with gloo
and world_size 2, that the schedule and the transports reproduce the oracle's
single-process SVD bit for bit.  Never used by the product path."""
import math

import numpy as np

import oracle as O
import paper_2202_08361_b200 as J


def _f64(x):
    return x.view(np.float64) if np.iscomplexobj(x) else x


def _flat(X):
    """float64 view of all of a Fortran-ordered real/complex matrix"""
    return _f64(X.reshape(-1, order="F"))


def _slot_position(B, P, rank, slot):
    i = rank * (B // 2 // P) + slot // 2
    return B - 1 - i if slot % 2 else i


def _owner(B, P, pos):
    per = B // 2 // P
    low = pos < B // 2
    i = pos if low else B - 1 - pos
    return i // per, 2 * (i % per) + (0 if low else 1)


def _Fm(cplx, m):
    k = m.bit_length() - 1
    return 1022 - k if not cplx else 1021 - k - (1 if m * m >= 1 << (2 * k + 1) else 0)


def _ilogb(x):
    return math.frexp(x)[1] - 1


def sharded_gesvj_model(A, nblocks, transport, R, max_sweeps=30, s0_adjust=0):
    """This rank's part of the sharded SVD of A (numpy m x n; every rank passes
    the whole A and keeps its columns).  Returns dict like J.gesvj plus U, V
    (local columns) and cols (their global indices)."""
    m, n = A.shape
    cplx = np.iscomplexobj(A)
    P, rank, B = transport.nranks, transport.rank, nblocks
    b = n // B
    cols = np.array(J.dist_columns(n, B, rank, P))
    nl = len(cols)
    nslots = nl // b
    G = np.asfortranarray(A[:, cols].copy())  # m x nl
    V = np.zeros((n, nl), dtype=A.dtype, order="F")
    V[cols, np.arange(nl)] = 1.0
    # line 1: global M0, s0
    w = np.array([np.frombuffer(np.float64(np.abs(_flat(G)).max()).tobytes(), np.int64)[0]])
    transport.allreduce(w, 0)
    M = float(np.frombuffer(w.tobytes(), np.float64)[0])
    F, K = _Fm(cplx, m), (1020 if cplx else 1022)
    s = F - _ilogb(M) - 1 + s0_adjust
    _flat(G)[...] = np.ldexp(_flat(G), s)
    Mt = math.ldexp(M, s)
    tps, converged, C = [], False, max_sweeps
    for c in range(max_sweeps):
        T = 0
        for k in range(n - 1):
            if O.strategy_is_checkpoint(n, B, k):  # Eq. (skr) on the global M-tilde
                w = np.array([np.frombuffer(np.float64(Mt).tobytes(), np.int64)[0]])
                transport.allreduce(w, 0)
                Mt = float(np.frombuffer(w.tobytes(), np.float64)[0])
                lm = _ilogb(Mt)
                if K - lm < 0:
                    sn = F - lm - 1
                    _flat(G)[...] = np.ldexp(_flat(G), sn)
                    Mt = math.ldexp(Mt, sn)
                    s += sn
            pairs = np.array(J.dist_local_pairs(n, B, rank, P, k), dtype=np.int32)
            out = O.step(G, V, pairs, R)
            T += out["t"]
            Mt = max(Mt, out["mmax"])
            if k >= b - 1 and (k - (b - 1)) % b == b - 1:  # end of a phase-II round
                G2, V2 = np.empty_like(G), np.empty_like(V)
                ops = []
                for sl in range(nslots):
                    pos = _slot_position(B, P, rank, sl)
                    dpos = 0 if pos == 0 else (pos - 1 if pos >= 2 else B - 1)
                    dr, ds = _owner(B, P, dpos)
                    if dr == rank:
                        G2[:, ds * b:(ds + 1) * b] = G[:, sl * b:(sl + 1) * b]
                        V2[:, ds * b:(ds + 1) * b] = V[:, sl * b:(sl + 1) * b]
                    else:
                        for X in (G, V):
                            blk = np.asfortranarray(X[:, sl * b:(sl + 1) * b])
                            ops.append((dr, 0, _f64(blk.reshape(-1, order="F")).view(np.uint8)))
                recv = []
                for ds in range(nslots):
                    dpos = _slot_position(B, P, rank, ds)
                    spos = 0 if dpos == 0 else (1 if dpos == B - 1 else dpos + 1)
                    sr, _ = _owner(B, P, spos)
                    if sr != rank:
                        for X in (G2, V2):
                            blk = np.empty((X.shape[0], b), dtype=X.dtype, order="F")
                            recv.append((X, ds, blk))
                            ops.append((sr, 1, _f64(blk.reshape(-1, order="F")).view(np.uint8)))
                transport.sendrecv(ops)
                for X, ds, blk in recv:
                    X[:, ds * b:(ds + 1) * b] = blk
                G, V = G2, V2
        w = np.array([T], dtype=np.int64)
        transport.allreduce(w, 1)
        T = int(w[0])
        tps.append(T)
        if T == 0:
            converged, C = True, c + 1
            break
    ef = [O.colnorm(np.ascontiguousarray(G[:, j]), R) for j in range(nl)]
    e = np.array([x for x, _ in ef])
    f = np.array([y for _, y in ef])
    if converged:
        for j in range(nl):
            if not math.isinf(e[j]):
                _f64(G[:, j])[...] = np.ldexp(_f64(G[:, j]), -int(e[j])) / f[j]
        ek = np.where(np.isinf(e), e, e - s)
    else:
        ek = e
    keys = np.stack([ek, f, cols.astype(np.float64)], 1).reshape(-1)
    allk = transport.allgather(keys.view(np.uint8)).view(np.float64).reshape(-1, 3)
    if converged:
        order = sorted(range(n), key=lambda j: (-allk[j, 0], -allk[j, 1], allk[j, 2]))
    else:
        order = list(np.argsort(allk[:, 2]))
    se, sf = allk[order, 0], allk[order, 1]
    sigma = np.array([0.0 if math.isinf(x) else math.ldexp(y, int(max(min(x, 1e5), -1e5)))
                      for x, y in zip(se, sf)])
    perm = allk[order, 2].astype(np.int64)
    return dict(U=G, V=V, cols=cols, sigma=sigma, sigma_e=se, sigma_f=sf, perm=perm, sweeps=C,
                tps=tps, status=0 if converged else 1, scale=s)
