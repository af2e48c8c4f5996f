"""Column-block-sharded jsvd_gesvj (BASELINE configs[4]): bootstrap and transports.

north_star: "A single large SVD splits by column blocks under a round-robin block
ordering, with blocks exchanged between steps by NCCL send/recv over NVLink."

Everything of the method runs inside libjsvd: jsvd_gesvj with a ``jsvd_dist``
(include/jsvd.h) generates this rank's pivot pairs of the block round-robin
(R#20, B = nblocks blocks) on the device, all-reduces M-tilde at
the Eq. (skr) check points and T per sweep, moves the column blocks of G and V
after every phase-II round (NCCL send/recv inside one group, on the caller's
stream), and finalizes (norms, normalisation, the global sort of sigma) in
its kernels.  The ordering and check schedule depend only on (n, nblocks), so
U, V, sigma are bit-identical for every number of ranks.

This module only builds the ``jsvd_dist`` a rank passes:
  NcclDist        the library's own NCCL communicator; the 128-byte unique id
                  is broadcast over a torch.distributed group (the bootstrap)
  GlooTransport   host-staged transport over a torch.distributed CPU group
                  (gloo): the library stages blocks through pinned host
                  buffers, the callbacks move the bytes between processes
  ThreadGroup     P ranks as threads of one process (host-staged through
                  shared memory), e.g. one thread per GPU, or P virtual ranks
                  on one GPU -- each rank's kernels run on its own stream and
                  never wait on another rank's kernels; the host rendezvous in
                  the callbacks is the only synchronisation
and maps a matrix's columns to ranks (``local_columns``).
"""
import ctypes as ct
import threading
import traceback

import numpy as np
import torch

import paper_2202_08361_b200 as J

__all__ = ["NcclDist", "GlooTransport", "ThreadGroup", "local_columns", "gesvj_sharded",
           "run_thread_ranks"]


def local_columns(n, nblocks, rank, nranks):
    """Global column indices of rank `rank`'s local columns, in local order
    (jsvd_dist_columns): scatter A[:, cols] to the rank, gather U the same way."""
    return np.array(J.dist_columns(n, nblocks, rank, nranks), dtype=np.int64)


def gesvj_sharded(A_local, n, nblocks, dist, **kw):
    """jsvd_gesvj on this rank's columns (A_local: m x n/nranks column-major CUDA
    tensor, packed).  Returns the dict of J.gesvj (sigma / perm global)."""
    return J.gesvj(A_local, nblocks=nblocks, dist=dist, n=n, **kw)


class _StdoutToStderr:
    """fd-level redirect of stdout to stderr (NCCL may print its version banner
    on stdout at communicator creation; stdout stays clean for callers that
    print machine-readable output, such as bench.py's JSON line)."""

    def __enter__(self):
        import os
        import sys
        sys.stdout.flush()
        self._saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *a):
        import os
        import sys
        sys.stdout.flush()
        os.dup2(self._saved, 1)
        os.close(self._saved)


class NcclDist:
    """The library's NCCL communicator for this process's rank of `group`
    (torch.distributed, any backend; only the unique id travels through it).
    ``.dist`` is the jsvd_dist to pass; close() destroys the communicator."""

    def __init__(self, group=None, flags=0):
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [J.nccl_unique_id() if rank == 0 else None]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(obj, src=src, group=group)
        with _StdoutToStderr():
            self.comm = J.nccl_comm_init(world, obj[0], rank)
        self.dist = J.Dist(self.comm, rank, world, None, flags)

    @classmethod
    def single(cls, flags=J.DIST_SELF_P2P):
        """A world of one rank (no torch.distributed needed): with
        DIST_SELF_P2P every block move goes through NCCL send/recv to self."""
        self = cls.__new__(cls)
        with _StdoutToStderr():
            self.comm = J.nccl_comm_init(1, J.nccl_unique_id(), 0)
        self.dist = J.Dist(self.comm, 0, 1, None, flags)
        return self

    def close(self):
        if self.comm:
            J.nccl_comm_destroy(self.comm)
            self.comm = None


def _u8(ptr, nbytes):
    return np.ctypeslib.as_array(ct.cast(ptr, ct.POINTER(ct.c_uint8)), (int(nbytes),))


class _HostTransport:
    """ctypes callbacks of jsvd_transport around three methods a subclass
    provides: sendrecv(ops) with ops [(peer, dir, uint8 array)], allreduce(words,
    op) on an int64 array in place (op 0 max, 1 sum), allgather(uint8 array) ->
    uint8 array of nranks * size.  Exceptions become a nonzero return."""

    def __init__(self, rank, nranks):
        self.rank, self.nranks = rank, nranks
        self._cb = (J.SENDRECV_FN(self._sr), J.ALLREDUCE_FN(self._ar), J.ALLGATHER_FN(self._ag))
        self.xport = J.Transport(None, *self._cb)
        self.dist = J.Dist(None, rank, nranks, ct.pointer(self.xport), 0)

    def _sr(self, ctx, nops, peer, dirs, buf, nbytes):
        try:
            self.sendrecv([(peer[k], dirs[k], _u8(buf[k], nbytes[k])) for k in range(nops)])
            return 0
        except Exception:
            traceback.print_exc()
            return 1

    def _ar(self, ctx, buf, count, op):
        try:
            # op 0 reduces bits of non-negative doubles (< 2^63): signed max is the same
            w = np.ctypeslib.as_array(ct.cast(buf, ct.POINTER(ct.c_int64)), (int(count),))
            self.allreduce(w, op)
            return 0
        except Exception:
            traceback.print_exc()
            return 1

    def _ag(self, ctx, send, recv, nbytes):
        try:
            out = self.allgather(_u8(send, nbytes).copy())
            _u8(recv, nbytes * self.nranks)[:] = out
            return 0
        except Exception:
            traceback.print_exc()
            return 1


class GlooTransport(_HostTransport):
    """Host-staged transport over a torch.distributed CPU group (gloo)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.d, self.group = dist, group
        super().__init__(dist.get_rank(group), dist.get_world_size(group))

    def _peer(self, r):
        return self.d.get_global_rank(self.group, r) if self.group is not None else r

    def sendrecv(self, ops):
        # the k-th operation to / from one peer matches the peer's k-th (the
        # library lists both sides by source circle position, G then V)
        seq, reqs = {}, []
        for peer, dirn, a in ops:
            tag = seq.get((peer, dirn), 0)
            seq[(peer, dirn)] = tag + 1
            t = torch.from_numpy(a)
            f = self.d.isend if dirn == 0 else self.d.irecv
            reqs.append(f(t, self._peer(peer), group=self.group, tag=tag))
        for r in reqs:
            r.wait()

    def allreduce(self, words, op):
        t = torch.from_numpy(words)
        self.d.all_reduce(t, op=self.d.ReduceOp.MAX if op == 0 else self.d.ReduceOp.SUM,
                          group=self.group)

    def allgather(self, a):
        parts = [torch.empty_like(torch.from_numpy(a)) for _ in range(self.nranks)]
        self.d.all_gather(parts, torch.from_numpy(a), group=self.group)
        return torch.cat(parts).numpy()


class ThreadGroup:
    """P ranks as threads of one process: host-staged collectives through
    shared memory, a barrier per collective.  transport(rank) gives each
    thread's jsvd_dist."""

    def __init__(self, P):
        self.P = P
        self.bar = threading.Barrier(P)
        self.box = {}
        self.lock = threading.Lock()

    def transport(self, rank):
        g = self

        class _T(_HostTransport):
            def sendrecv(self, ops):
                seq = {}
                for peer, dirn, a in ops:
                    k = seq.get((peer, dirn), 0)
                    seq[(peer, dirn)] = k + 1
                    if dirn == 0:
                        with g.lock:
                            g.box[(self.rank, peer, k)] = a.copy()
                g.bar.wait()
                seq = {}
                for peer, dirn, a in ops:
                    k = seq.get((peer, dirn), 0)
                    seq[(peer, dirn)] = k + 1
                    if dirn == 1:
                        with g.lock:
                            a[:] = g.box.pop((peer, self.rank, k))
                g.bar.wait()

            def allreduce(self, words, op):
                with g.lock:
                    g.box[("ar", self.rank)] = words.copy()
                g.bar.wait()
                allw = [g.box[("ar", r)] for r in range(g.P)]
                words[:] = np.max(allw, axis=0) if op == 0 else np.sum(allw, axis=0)
                g.bar.wait()
                if self.rank == 0:
                    for r in range(g.P):
                        g.box.pop(("ar", r))
                g.bar.wait()

            def allgather(self, a):
                with g.lock:
                    g.box[("ag", self.rank)] = a
                g.bar.wait()
                out = np.concatenate([g.box[("ag", r)] for r in range(g.P)])
                g.bar.wait()
                if self.rank == 0:
                    for r in range(g.P):
                        g.box.pop(("ag", r))
                g.bar.wait()
                return out

        return _T(rank, self.P)


def run_thread_ranks(A, nblocks, P, max_sweeps=30, device=None, s0_adjust=0):
    """The sharded SVD of A (numpy m x n, or a CUDA tensor) as P thread ranks
    on the current device (each on its own stream).  Returns (results per
    rank, local column indices per rank)."""
    m, n = A.shape
    At = torch.as_tensor(A)
    g = ThreadGroup(P)
    outs, errs = [None] * P, []
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    cols = [local_columns(n, nblocks, r, P) for r in range(P)]
    parts = [At[:, c].T.contiguous().to(dev).T for c in cols]  # m x n/P column-major, packed
    torch.cuda.synchronize(dev)

    def run(r):
        try:
            torch.cuda.set_device(dev)
            s = torch.cuda.Stream(dev)
            tr = g.transport(r)
            with torch.cuda.stream(s):
                outs[r] = gesvj_sharded(parts[r], n, nblocks, tr.dist, max_sweeps=max_sweeps,
                                        stream=s, s0_adjust=s0_adjust)
            s.synchronize()
            outs[r]["_transport"] = tr
        except Exception as e:  # surfaced by the caller
            errs.append(e)
            g.bar.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return outs, cols
