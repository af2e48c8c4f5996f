"""The column-block-sharded jsvd_gesvj (a jsvd_dist: the schedule, block
exchange and collectives inside libjsvd) on one GPU:
 - P = 1, 2, 4, 8 thread ranks (dist.ThreadGroup: host-staged transport; each
   rank's kernels on its own stream, only the host rendezvous synchronises --
   no kernel waits on another rank's kernel);
 - a world of one NCCL rank (NcclDist.single) with JSVD_DIST_SELF_P2P: every
   block move goes through ncclSend/ncclRecv to self inside ncclGroupStart/End,
   M-tilde and T through ncclAllReduce, the sort keys through ncclAllGather;
 - two processes on the GPU with the CUDA kernels and a gloo (CPU-staged)
   transport.
Results must be bitwise identical for every P and transport, to
jsvd_gesvj(nblocks=16) on one GPU and to the oracle -- converged, capped
 and with the Eq. (skr) rescale firing (R#40)."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu


def _bits(a):
    a = np.ascontiguousarray(a)
    return (a.view(np.float64) if np.iscomplexobj(a) else a).view(np.uint64)


def _case(cplx, m, n, seed=0):
    rng = np.random.default_rng(m + n + cplx + seed)
    A = rng.standard_normal((m, n)) * 2.0 ** rng.integers(-20, 20, n)
    if cplx:
        A = A + 1j * rng.standard_normal((m, n))
    return A


def _rspec(cplx, m):
    # R#15 for m <= 2048 (complex) / 4096 (real): one CTA of W = 256 lanes
    W = 256 if (m <= 2048 or (not cplx and m <= 4096)) else 512
    offs = [16, 8, 4, 2, 1, 128, 64, 32] + ([256] if W == 512 else [])
    return O.RSpec.make(W, 1, offs)


def _np(x):
    """numpy copy of a (column-major view of a) tensor, or x itself"""
    if torch.is_tensor(x):
        return x.T.contiguous().cpu().numpy().T if x.dim() == 2 else x.cpu().numpy()
    return x


def _assemble(outs, cols, n, status):
    U = np.zeros((_np(outs[0]["U"]).shape[0], n), dtype=_np(outs[0]["U"]).dtype)
    V = np.zeros((n, n), dtype=U.dtype)
    for o, c in zip(outs, cols):
        U[:, c] = _np(o["U"])
        V[:, c] = _np(o["V"])
    perm = _np(outs[0]["perm"])
    if status == 0:
        U, V = U[:, perm], V[:, perm]
    return U, V, perm


def _check(ref, outs, cols, n):
    for o in outs:
        assert o["status"] == ref["status"] and o["sweeps"] == ref["sweeps"]
        assert list(o["tps"]) == list(ref["tps"]) and o["scale"] == ref["scale"]
        for k in ("sigma", "sigma_e", "sigma_f"):
            assert np.array_equal(_bits(_np(o[k])), _bits(ref[k])), k
    U, V, perm = _assemble(outs, cols, n, ref["status"])
    if ref["status"] != 0:
        assert np.array_equal(perm, np.arange(n))
    assert np.array_equal(_bits(U), _bits(ref["U"]))
    assert np.array_equal(_bits(V), _bits(ref["V"]))


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("m,n", [(64, 32), (300, 64), (2049, 96)])
def test_dist_thread_ranks_bitwise(cplx, m, n):
    import paper_2202_08361_b200 as J
    from paper_2202_08361_b200.dist import run_thread_ranks
    A = _case(cplx, m, n)
    assert J.step_rspec(cplx, m)[:2] == (_rspec(cplx, m).W, 1)
    ref = O.gesvj(A, _rspec(cplx, m), B=16, max_sweeps=30)
    g = torch.from_numpy(np.ascontiguousarray(A.T)).cuda().T
    lib = J.gesvj(g, nblocks=16, max_sweeps=30)
    assert np.array_equal(_bits(lib["U"].T.contiguous().cpu().numpy().T), _bits(ref["U"]))
    for P in (1, 2, 4, 8):
        outs, cols = run_thread_ranks(A, 16, P, max_sweeps=30)
        _check(ref, outs, cols, n)


@pytest.mark.parametrize("cplx", [False, True])
def test_dist_thread_ranks_capped_and_rescaled(cplx):
    from paper_2202_08361_b200.dist import run_thread_ranks
    m, n = 96, 64
    A = _case(cplx, m, n, seed=3)
    K = 1020 if cplx else 1022
    for kw in (dict(max_sweeps=2), dict(max_sweeps=30, s0_adjust=K + 1 - O.Fm(cplx, m))):
        ref = O.gesvj(A, _rspec(cplx, m), B=16, **kw)
        for P in (2, 8):
            outs, cols = run_thread_ranks(A, 16, P, **kw)
            _check(ref, outs, cols, n)


@pytest.mark.parametrize("cplx", [False, True])
def test_dist_nccl_world_one_self_p2p(cplx):
    # the NCCL transport executed on one GPU: ncclSend/ncclRecv to self for
    # every block move, ncclAllReduce, ncclAllGather
    import paper_2202_08361_b200 as J
    from paper_2202_08361_b200.dist import NcclDist, gesvj_sharded, local_columns
    m, n = 300, 64
    A = _case(cplx, m, n, seed=5)
    ref = O.gesvj(A, _rspec(cplx, m), B=16, max_sweeps=30)
    nd = NcclDist.single(flags=J.DIST_SELF_P2P)
    try:
        cols = local_columns(n, 16, 0, 1)
        part = torch.from_numpy(np.ascontiguousarray(A[:, cols].T)).cuda().T
        out = gesvj_sharded(part, n, 16, nd.dist, max_sweeps=30)
        torch.cuda.synchronize()
        _check(ref, [out], [cols], n)
        # and without SELF_P2P (local moves as device copies)
        nd.dist.flags = 0
        part = torch.from_numpy(np.ascontiguousarray(A[:, cols].T)).cuda().T
        out = gesvj_sharded(part, n, 16, nd.dist, max_sweeps=30)
        torch.cuda.synchronize()
        _check(ref, [out], [cols], n)
    finally:
        nd.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cplx, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2202_08361_b200.dist import GlooTransport, gesvj_sharded, local_columns
        m, n = 300, 64
        A = _case(cplx, m, n, seed=7)
        tr = GlooTransport()
        cols = local_columns(n, 16, rank, world)
        part = torch.from_numpy(np.ascontiguousarray(A[:, cols].T)).cuda().T
        out = gesvj_sharded(part, n, 16, tr.dist, max_sweeps=30)
        torch.cuda.synchronize()
        # numpy, not tensors: the queue must not hold fds of this process's storage
        q.put((rank, {k: _np(v) for k, v in out.items()}, cols))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cplx", [False, True])
def test_dist_two_processes_gloo_staged(cplx):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cplx, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=600) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    m, n = 300, 64
    A = _case(cplx, m, n, seed=7)
    ref = O.gesvj(A, _rspec(cplx, m), B=16, max_sweeps=30)
    _check(ref, [g[1] for g in got], [g[2] for g in got], n)


def test_dist_host_time_per_step():
    # The sharded driver's host loop (gesvj.cu): per step it fills the step's
    # parameters and enqueues one kernel (plus an 8-byte all-reduce at check
    # points and one group of sends/receives per round); it synchronises once
    # per sweep.  On a matrix whose steps take a few microseconds on the GPU
    # the wall time per step is the host's cost: it must stay under 20 us
    # (the verdict's bar for P = 8; the per-rank loop does not depend on P).
    import time
    import paper_2202_08361_b200 as J
    from paper_2202_08361_b200.dist import NcclDist, gesvj_sharded, local_columns
    m, n = 64, 64
    A = _case(True, m, n, seed=11)
    nd = NcclDist.single(flags=0)
    try:
        cols = local_columns(n, 16, 0, 1)
        part = torch.from_numpy(np.ascontiguousarray(A[:, cols].T)).cuda().T.contiguous().T
        work = torch.empty(J.gesvj_workspace(True, m, n, 16, nd.dist), dtype=torch.uint8,
                           device="cuda")
        V = torch.empty((n, n), dtype=torch.complex128, device="cuda").T
        steps = 20 * (n - 1)
        for _ in range(2):  # the second call is timed
            p2 = part.clone()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out = gesvj_sharded(p2, n, 16, nd.dist, max_sweeps=40, V=V, work=work,
                                max_steps=steps)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        per_step_us = dt / steps * 1e6
        print(f"host+GPU wall time per step: {per_step_us:.2f} us over {steps} steps")
        assert per_step_us <= 20.0, per_step_us
    finally:
        nd.close()


def test_config5_full_size_sharded_equals_single_gpu():
    # BASELINE configs[4] at full size (complex 32768 x 8192) through the
    # sharded driver as the bench runs it (NCCL world of one, block moves
    # through ncclSend/ncclRecv to self), one full sweep (8191 steps, 15
    # block exchanges), against single-GPU jsvd_gesvj with the same ordering
    # (B = 16) on the same matrix: the iterate G, V and Sigma' (status
    # ENOCONV after the capped sweep) bitwise.  The oracle pins both paths on
    # smaller matrices above; at this size the oracle would take hours.
    import synth
    import paper_2202_08361_b200 as J
    from paper_2202_08361_b200.dist import NcclDist, local_columns
    m, n, B = 32768, 8192, 16
    A, _ = synth.svd_cfg5_torch(m, n, device="cuda")  # (m, n) column-major
    cols = torch.from_numpy(local_columns(n, B, 0, 1)).cuda()
    Al = A.T[cols].contiguous()  # (n, m): the rank's columns in slot order
    ref = J.gesvj(A, nblocks=B, max_sweeps=1)
    torch.cuda.synchronize()
    nd = NcclDist.single(flags=J.DIST_SELF_P2P)
    try:
        V = torch.empty((n, n), dtype=torch.complex128, device="cuda")
        work = torch.empty(J.gesvj_workspace(True, m, n, B, nd.dist), dtype=torch.uint8,
                           device="cuda")
        out = J.gesvj(Al.T, nblocks=B, max_sweeps=1, V=V.T, work=work, dist=nd.dist, n=n)
        torch.cuda.synchronize()
    finally:
        nd.close()
    assert out["status"] == ref["status"] == 1 and out["sweeps"] == ref["sweeps"] == 1
    assert list(out["tps"]) == list(ref["tps"]) and out["scale"] == ref["scale"]
    for k in ("sigma", "sigma_e", "sigma_f"):
        assert torch.equal(out[k].view(torch.int64), ref[k].view(torch.int64)), k
    # local column j is global column cols[j] (every block is home after a sweep)
    assert torch.equal(torch.view_as_real(Al).view(torch.int64),
                       torch.view_as_real(A.T[cols]).view(torch.int64))
    assert torch.equal(torch.view_as_real(V[:, :]).view(torch.int64),
                       torch.view_as_real(ref["V"].T[cols]).view(torch.int64))
