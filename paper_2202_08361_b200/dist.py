"""Column-block-sharded one-sided Jacobi SVD (BASELINE configs[4]).

north_star: "A single large SVD splits by column blocks under a round-robin block
ordering, with blocks exchanged between steps by NCCL send/recv over NVLink."

The iteration is Alg 4.1 with the block round-robin ordering of
DESIGN.md R#20 on B = 16 column blocks of b = n/B columns:
  phase I   b-1 steps of flat round-robin inside every block (local to a rank);
  phase II  B-1 rounds; in round r the circle method on the 16 blocks gives 8
            block pairs, each rank owns 8/P of them; step t of the round pairs
            column j of the lower block with column (j+t) mod b of the higher;
            after the round every block moves one circle position
            (position k -> k-1, position 1 -> B-1, position 0 fixed): at most
            two blocks of G and of V leave and arrive per rank (NCCL send/recv).
The rescale check (Eq. skr) runs at phase I's start and at every round's start
on the GLOBAL M-tilde (all-reduce max), T is summed per sweep (all-reduce sum):
the ordering and the check schedule depend only on (n, B), so U, V, sigma are
bit-identical for P = 1, 2, 4, 8 and to jsvd_gesvj / the oracle with nblocks=16.

This module is host scheduling only.  Every arithmetic step runs in the
library's kernels (CudaCompute: jsvd_sweep_step, jsvd_maxnorm, jsvd_scale,
jsvd_colnorms, jsvd_normalize); the collectives are torch.distributed (NCCL
over NVLink on a B200 box).  The rank and compute objects are pluggable so the
same schedule runs as P real ranks (TorchDistRanks), as P virtual ranks in one
process on one GPU (LocalRanks: copies instead of messages -- no kernel ever
waits on another), and, in the CPU test suite only, with a test-supplied
compute object.
"""
import math

import numpy as np
import torch

__all__ = ["BlockSchedule", "LocalRanks", "TorchDistRanks", "CudaCompute", "DistJacobi", "gesvj_dist",
           "scatter_columns", "gather_columns", "Fm", "Kr"]


def Fm(cplx, m):
    """floor(lg(omega/(2m))) / floor(lg(omega/(4 m sqrt2))) in exact integers (R#28)."""
    k = m.bit_length() - 1
    if not cplx:
        return 1022 - k
    return 1021 - k - (1 if m * m >= 1 << (2 * k + 1) else 0)


def Kr(cplx):
    return 1020 if cplx else 1022


def _ilogb(x):
    return math.frexp(x)[1] - 1  # floor(lg x) for finite x > 0


class BlockSchedule:
    """The block round-robin ordering over P ranks (R#20)."""

    def __init__(self, n, B=16, P=1):
        if n % B or B % 2 or (B // 2) % P:
            raise ValueError("need B | n, B even and P | B/2")
        self.n, self.B, self.P, self.b = n, B, P, n // B
        if self.b > 1 and self.b % 2:
            raise ValueError("n/B must be even")
        self.per = (B // 2) // P  # block pairs per rank
        self.nslots = 2 * self.per

    # circle method on B players
    def block_at(self, r, pos):
        return 0 if pos == 0 else ((pos - 1 + r) % (self.B - 1)) + 1

    def owner(self, pos):
        """(rank, slot) holding circle position pos."""
        i = pos if pos < self.B // 2 else self.B - 1 - pos
        return i // self.per, 2 * (i % self.per) + (0 if pos < self.B // 2 else 1)

    def slot_position(self, rank, slot):
        i = rank * self.per + slot // 2
        return i if slot % 2 == 0 else self.B - 1 - i

    def local_block(self, rank, slot, r):
        return self.block_at(r, self.slot_position(rank, slot))

    def steps_per_sweep(self):
        return self.n - 1

    def is_checkpoint(self, k):
        b = self.b
        if k == 0:
            return True
        if k < b - 1:
            return False
        return (k - (b - 1)) % b == 0

    def local_pairs(self, rank, k):
        """Pairs (local column indices, p < q by GLOBAL index) of step k in [0, n-1)."""
        b, out = self.b, []
        if k < b - 1:  # phase I: positions of round 0
            for slot in range(self.nslots):
                for i in range(b // 2):
                    x = 0 if i == 0 else ((i - 1 + k) % (b - 1)) + 1
                    yp = b - 1 - i
                    y = 0 if yp == 0 else ((yp - 1 + k) % (b - 1)) + 1
                    x, y = min(x, y), max(x, y)
                    out.append((slot * b + x, slot * b + y))
        else:
            s2 = k - (b - 1)
            r, t = s2 // b, s2 % b
            for kk in range(self.per):
                u, v = self.local_block(rank, 2 * kk, r), self.local_block(rank, 2 * kk + 1, r)
                lo, hi = (2 * kk, 2 * kk + 1) if u < v else (2 * kk + 1, 2 * kk)
                for j in range(b):
                    out.append((lo * b + j, hi * b + (j + t) % b))
        return np.array(out, dtype=np.int32).reshape(-1, 2)

    def global_pairs(self, rank, k):
        """The same pairs in global column indices (for checks against the oracle)."""
        r = 0 if k < self.b - 1 else (k - (self.b - 1)) // self.b
        loc = self.local_pairs(rank, k)
        g = lambda c: self.local_block(rank, c // self.b, r) * self.b + c % self.b
        return np.array([[g(p), g(q)] for p, q in loc], dtype=np.int32).reshape(-1, 2)

    def moves(self):
        """Block moves after a round: list of (src_rank, src_slot, dst_rank, dst_slot);
        position 0 stays (listed too: the exchange writes into a second buffer)."""
        out = [(*self.owner(0), *self.owner(0))]
        for pos in range(1, self.B):
            dst = pos - 1 if pos >= 2 else self.B - 1
            out.append((*self.owner(pos), *self.owner(dst)))
        return out


# --------------------------------------------------------------- rank backends
class LocalRanks:
    """P virtual ranks in one process (one GPU): collectives are local
    reductions, block messages are device copies; ranks run one after another
    (no kernel waits on another)."""

    def __init__(self, P):
        self.P, self.ranks = P, list(range(P))

    def allreduce_max(self, xs):
        m = torch.stack([x.reshape(()) for x in xs]).max()
        for x in xs:
            x.fill_(m.item())

    def allreduce_sum(self, xs):
        s = torch.stack([x.reshape(()) for x in xs]).sum()
        for x in xs:
            x.fill_(s.item())

    def allgather_cat(self, xs):
        return [torch.cat(xs)] * len(xs)

    def exchange(self, moves, bufs_src, bufs_dst, b):
        for sr, ss, dr, ds in moves:
            for src, dst in zip(bufs_src, bufs_dst):
                dst[dr][ds * b:(ds + 1) * b].copy_(src[sr][ss * b:(ss + 1) * b])


class TorchDistRanks:
    """One real rank per process over torch.distributed (NCCL on B200 boxes,
    gloo in the CPU tests)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.P = dist.get_world_size(group)
        self.ranks = [dist.get_rank(group)]

    def allreduce_max(self, xs):
        self.dist.all_reduce(xs[0], op=self.dist.ReduceOp.MAX, group=self.group)

    def allreduce_sum(self, xs):
        self.dist.all_reduce(xs[0], op=self.dist.ReduceOp.SUM, group=self.group)

    def allgather_cat(self, xs):
        parts = [torch.empty_like(xs[0]) for _ in range(self.P)]
        self.dist.all_gather(parts, xs[0].contiguous(), group=self.group)
        return [torch.cat(parts)]

    def exchange(self, moves, bufs_src, bufs_dst, b):
        me = self.ranks[0]
        nccl = self.dist.get_backend(self.group) == "nccl"
        ops, reqs = [], []
        for sr, ss, dr, ds in moves:
            for src, dst in zip(bufs_src, bufs_dst):
                blk_s, blk_d = src[0][ss * b:(ss + 1) * b], dst[0][ds * b:(ds + 1) * b]
                if sr == me and dr == me:
                    blk_d.copy_(blk_s)
                elif sr == me:
                    if nccl:
                        ops.append(self.dist.P2POp(self.dist.isend, blk_s, dr, group=self.group))
                    else:
                        reqs.append(self.dist.isend(blk_s, dr, group=self.group))
                elif dr == me:
                    if nccl:
                        ops.append(self.dist.P2POp(self.dist.irecv, blk_d, sr, group=self.group))
                    else:
                        reqs.append(self.dist.irecv(blk_d, sr, group=self.group))
        if ops:  # NCCL: one group of sends/receives over NVLink
            reqs += self.dist.batch_isend_irecv(ops)
        for req in reqs:
            req.wait()


# --------------------------------------------------------------- compute
class CudaCompute:
    """The library's kernels on column-major CUDA tensors (storage: Gt of shape
    (ncols, m), i.e. G = Gt.T column-major)."""

    def __init__(self):
        import paper_2202_08361_b200 as J
        self.J = J
        self._pairs = {}

    def scalar(self, v, like):
        return torch.full((1,), float(v), dtype=torch.float64, device=like.device)

    def counter(self, like):
        return torch.zeros(1, dtype=torch.int64, device=like.device)

    def maxnorm(self, Gt, out):
        self.J.maxnorm(Gt.T, out=out)

    def scale(self, Gt, s):
        self.J.scale(Gt.T, s)

    def step(self, Gt, Vt, pairs, key, t_dev, mt_dev, ce, cf):
        dev = self._pairs.get(key)
        if dev is None:
            dev = torch.from_numpy(pairs).to(Gt.device)
            self._pairs[key] = dev
        self.J.sweep_step(Gt.T, Vt.T, dev, col_e=ce, col_f=cf, t_dev=t_dev, mmax_dev=mt_dev)

    def colnorms(self, Gt):
        return self.J.colnorms(Gt.T)

    def normalize(self, Gt, ce, cf):
        self.J.normalize(Gt.T, ce, cf)


def scatter_columns(A, sched, rank):
    """The round-0 local column blocks of rank `rank` as Gt (ncols, m) row-major."""
    b = sched.b
    blocks = [sched.local_block(rank, s, 0) for s in range(sched.nslots)]
    cols = np.concatenate([np.arange(bl * b, (bl + 1) * b) for bl in blocks])
    return cols


def gather_columns(parts, sched):
    """Inverse of scatter_columns: list over ranks of (ncols_local, rows) -> (n, rows)."""
    b = sched.b
    out = [None] * sched.n
    for rank, part in enumerate(parts):
        for s in range(sched.nslots):
            bl = sched.local_block(rank, s, 0)
            for j in range(b):
                out[bl * b + j] = part[s * b + j]
    return out


class DistJacobi:
    """Alg 4.1 on column blocks, step by step (gesvj_dist drives it to the end;
    bench.py times its steps).

    Gts: list (one per local rank of `ranks`) of Gt tensors (ncols_local, m)
    holding the round-0 column blocks (see scatter_columns).
    """

    def __init__(self, Gts, sched, ranks, compute, cplx=False):
        self.sched, self.ranks, self.compute, self.cplx = sched, ranks, compute, cplx
        nl = len(ranks.ranks)
        self.m = Gts[0].shape[1]
        like = Gts[0]
        # ---- line 1: M0 (global), s0, G1 = 2^s0 G
        self.Mt = [compute.scalar(0.0, like) for _ in range(nl)]
        for G, M in zip(Gts, self.Mt):
            compute.maxnorm(G, M)
        ranks.allreduce_max(self.Mt)
        M0 = float(self.Mt[0].item())
        if math.isinf(M0) or math.isnan(M0):
            raise ValueError("non-finite input (P:1112)")
        if M0 == 0.0:
            raise ValueError("zero matrix (P:1114)")
        self.F, self.K = Fm(cplx, self.m), Kr(cplx)
        self.s = self.F - _ilogb(M0) - 1
        for G in Gts:
            compute.scale(G, self.s)
        for M in self.Mt:
            M.fill_(math.ldexp(M0, self.s))
        # ---- line 2: V = I (local columns)
        self.Gts, self.Vts = Gts, []
        for rank, G in zip(ranks.ranks, Gts):
            cols = scatter_columns(None, sched, rank)
            V = torch.zeros((len(cols), sched.n), dtype=G.dtype, device=G.device)
            V[torch.arange(len(cols)), torch.from_numpy(cols).to(G.device)] = 1.0
            self.Vts.append(V)
        self.Gb = [torch.empty_like(G) for G in Gts]
        self.Vb = [torch.empty_like(V) for V in self.Vts]
        self.tdev = [compute.counter(like) for _ in range(nl)]
        self.ce = [torch.empty(G.shape[0], dtype=torch.float64, device=G.device) for G in Gts]
        self.cf = [torch.empty(G.shape[0], dtype=torch.float64, device=G.device) for G in Gts]
        self.moves = sched.moves()

    def begin_sweep(self):
        for t in self.tdev:
            t.zero_()

    def step(self, k):
        """Step k in [0, n-1) of the current sweep, incl. its check point and,
        at the end of a phase-II round, the block exchange."""
        S, b = self.sched, self.sched.b
        if S.is_checkpoint(k):  # Eq. (skr) on the global M-tilde (R#21)
            self.ranks.allreduce_max(self.Mt)
            mt = float(self.Mt[0].item())
            lm = _ilogb(mt)
            if self.K - lm < 0:
                sn = self.F - lm - 1
                for G in self.Gts:
                    self.compute.scale(G, sn)
                for M in self.Mt:
                    M.fill_(math.ldexp(mt, sn))
                self.s += sn
        for rank, G, V, t, M, e, f in zip(self.ranks.ranks, self.Gts, self.Vts, self.tdev,
                                          self.Mt, self.ce, self.cf):
            self.compute.step(G, V, S.local_pairs(rank, k), (rank, k), t, M, e, f)
        if k >= b - 1 and (k - (b - 1)) % b == b - 1:  # end of a phase-II round
            self.ranks.exchange(self.moves, [self.Gts, self.Vts], [self.Gb, self.Vb], b)
            self.Gts, self.Gb = self.Gb, self.Gts
            self.Vts, self.Vb = self.Vb, self.Vts

    def end_sweep(self):
        self.ranks.allreduce_sum(self.tdev)
        return int(self.tdev[0].item())

    def finalize(self):
        """P:1473-1485 (R#23, R#24): local norms, normalise, global sort."""
        S, n = self.sched, self.sched.n
        keys = []
        for rank, G in zip(self.ranks.ranks, self.Gts):
            e, f = self.compute.colnorms(G)
            self.compute.normalize(G, e, f)
            gcol = torch.from_numpy(scatter_columns(None, S, rank)).to(torch.float64).to(e.device)
            keys.append(torch.stack([e, f, gcol], 1))
        allk = self.ranks.allgather_cat(keys)[0].cpu().numpy()
        e_all = np.where(np.isinf(allk[:, 0]), allk[:, 0], allk[:, 0] - self.s)
        order = sorted(range(n), key=lambda j: (-e_all[j], -allk[j, 1], allk[j, 2]))
        sig_e = e_all[order]
        sig_f = allk[order, 1]
        sigma = np.array([0.0 if math.isinf(e) else math.ldexp(f, int(max(min(e, 1e5), -1e5)))
                          for e, f in zip(sig_e, sig_f)])
        perm = allk[order, 2].astype(np.int64)
        return dict(Gts=self.Gts, Vts=self.Vts, sigma=sigma, sigma_e=sig_e, sigma_f=sig_f,
                    perm=perm)


def gesvj_dist(Gts, sched, ranks, compute, max_sweeps=30, cplx=False):
    """Run Alg 4.1 on column blocks to convergence.

    On exit the returned dict has Gts (U's columns, same layout as the input),
    Vts (local V columns), the globally sorted sigma / sigma_e / sigma_f, the
    permutation `perm` (global column index of each sorted singular value),
    sweeps, tps (T per sweep) and status (0, or 1 = ENOCONV).
    """
    D = DistJacobi(Gts, sched, ranks, compute, cplx)
    tps, converged, C = [], False, max_sweeps
    for c in range(max_sweeps):
        D.begin_sweep()
        for k in range(sched.n - 1):
            D.step(k)
        T = D.end_sweep()
        tps.append(T)
        if T == 0:
            converged, C = True, c + 1
            break
    out = D.finalize()
    out.update(sweeps=C, tps=tps, status=0 if converged else 1)
    return out
