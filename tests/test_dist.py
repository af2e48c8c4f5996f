"""The column-block-sharded SVD on CPU (no GPU):
 - the library's host-only schedule functions (jsvd_dist_columns,
   jsvd_dist_local_pairs -- the functions the step kernel evaluates on the
   device) against the oracle's block round-robin (R#20);
 - the host-staged transports of paper_2202_08361_b200.dist (ThreadGroup;
   GlooTransport over a world_size-2 gloo group), called through their ctypes
   callbacks exactly as libjsvd calls them;
 - a CPU model of the sharded driver (tests/dist_model.py: the library's
   pair schedule, the block moves, global check points, oracle compute) over
   those transports, BITWISE identical to the oracle's single-process SVD
   with the same ordering (nblocks = 16) for P = 1, 2, 4 thread ranks and a
   world_size-2 gloo run."""
import ctypes as ct
import os
import socket
import threading

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import paper_2202_08361_b200 as J
from paper_2202_08361_b200.dist import GlooTransport, ThreadGroup, local_columns


def _circle(P, r, pos):  # R#20 restated: position 0 fixed, the others rotate
    return 0 if pos == 0 else ((pos - 1 + r) % (P - 1)) + 1


def _global_of_local(n, B, P, rank, k, l):
    """global column of local column l on rank `rank` during step k: slot ->
    circle position -> block in the step's round -> column"""
    b = n // B
    per = B // 2 // P
    slot, j = l // b, l % b
    i = rank * per + slot // 2
    pos = B - 1 - i if slot % 2 else i
    r = 0 if k < b - 1 else (k - (b - 1)) // b
    return _circle(B, r, pos) * b + j


@pytest.mark.parametrize("n", [32, 64, 96, 128])
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_local_pairs_are_the_oracle_block_round_robin(n, P):
    B = 16
    for rank in range(P):  # round 0 columns
        cols = J.dist_columns(n, B, rank, P)
        assert cols == [_global_of_local(n, B, P, rank, 0, l) for l in range(n // P)]
    for k in range(n - 1):
        got = []
        for rank in range(P):
            loc = J.dist_local_pairs(n, B, rank, P, k)
            flat = [x for pq in loc for x in pq]
            assert len(set(flat)) == len(flat) and max(flat) < n // P
            got += [(_global_of_local(n, B, P, rank, k, p), _global_of_local(n, B, P, rank, k, q))
                    for p, q in loc]
        ref = [tuple(x) for x in O.strategy_pairs(n, B, k).tolist()]
        # the same ordered pairs (p < q globally: the rotation is not symmetric)
        assert sorted(got) == sorted(ref), k


def test_dist_schedule_rejects_bad_arguments():
    with pytest.raises(J.JsvdError):
        J.dist_columns(64, 16, 0, 3)     # 3 does not divide B/2
    with pytest.raises(J.JsvdError):
        J.dist_columns(64, 64, 0, 1)     # flat RR (B = n) is not a block ordering
    with pytest.raises(J.JsvdError):
        J.dist_local_pairs(64, 16, 2, 2, 0)  # rank out of range
    with pytest.raises(J.JsvdError):
        J.dist_local_pairs(64, 16, 0, 2, 63)  # step out of range


def _case(cplx, m=64, n=32, seed=5):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, n)) * 2.0 ** rng.integers(-10, 10, n)
    if cplx:
        A = A + 1j * rng.standard_normal((m, n))
    return A


def _rspec(cplx, m):
    return O.RSpec.make(*J.step_rspec(cplx, m))  # host-only query


def _bits(a):
    a = np.ascontiguousarray(a)
    return (a.view(np.float64) if np.iscomplexobj(a) else a).view(np.uint64)


def _check_against_oracle(A, cplx, parts, res, max_sweeps=30, s0_adjust=0):
    n = A.shape[1]
    ref = O.gesvj(A, _rspec(cplx, A.shape[0]), B=16, max_sweeps=max_sweeps, s0_adjust=s0_adjust)
    U = np.zeros_like(ref["U"])
    V = np.zeros_like(ref["V"])
    for cols, Ul, Vl in parts:
        U[:, cols] = Ul
        V[:, cols] = Vl
    assert res["sweeps"] == ref["sweeps"] and res["status"] == ref["status"]
    assert list(res["tps"]) == list(ref["tps"]) and res["scale"] == ref["scale"]
    perm = np.asarray(res["perm"])
    if ref["status"] == 0:  # the oracle permutes U, V into sigma's order
        U, V = U[:, perm], V[:, perm]
    else:
        assert np.array_equal(perm, np.arange(n))
    for got, exp in ((U, ref["U"]), (V, ref["V"]), (res["sigma"], ref["sigma"]),
                     (res["sigma_e"], ref["sigma_e"]), (res["sigma_f"], ref["sigma_f"])):
        assert np.array_equal(_bits(got), _bits(exp))


def _run_threads(A, P, **kw):
    from dist_model import sharded_gesvj_model
    g = ThreadGroup(P)
    outs, errs = [None] * P, []

    def run(r):
        try:
            outs[r] = sharded_gesvj_model(A, 16, g.transport(r), _rspec(np.iscomplexobj(A), A.shape[0]), **kw)
        except Exception as e:
            errs.append(e)
            g.bar.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    return outs


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("P", [1, 2, 4])
def test_thread_ranks_model_bitwise(cplx, P):
    A = _case(cplx)
    outs = _run_threads(A, P)
    for o in outs[1:]:
        assert np.array_equal(_bits(o["sigma"]), _bits(outs[0]["sigma"]))
    _check_against_oracle(A, cplx, [(o["cols"], o["U"], o["V"]) for o in outs], outs[0])


@pytest.mark.parametrize("cplx", [False, True])
def test_thread_ranks_model_capped_and_rescaled(cplx):
    # P:1587-1593 (not converged: G = U Sigma', Sigma' in column order) and the
    # Eq. (skr) rescale firing in mid-run (R#40) through the sharded schedule
    A = _case(cplx, seed=9)
    adj = (1021 if cplx else 1023) - O.Fm(cplx, A.shape[0])
    for kw in (dict(max_sweeps=2), dict(s0_adjust=adj)):
        outs = _run_threads(A, 2, **kw)
        _check_against_oracle(A, cplx, [(o["cols"], o["U"], o["V"]) for o in outs], outs[0], **kw)


def test_thread_group_callbacks_through_ctypes():
    # the transport exactly as libjsvd calls it: C function pointers, host buffers
    P = 3
    g = ThreadGroup(P)
    res, errs = [None] * P, []

    def run(r):
        try:
            t = g.transport(r)
            x = t.xport
            w = (ct.c_int64 * 2)(10 * r + 1, -r)
            assert x.allreduce(None, ct.cast(w, ct.c_void_p), 2, 0) == 0
            v = (ct.c_int64 * 1)(r + 1)
            assert x.allreduce(None, ct.cast(v, ct.c_void_p), 1, 1) == 0
            snd = (ct.c_uint8 * 4)(*[r] * 4)
            rcv = (ct.c_uint8 * (4 * P))()
            assert x.allgather(None, ct.cast(snd, ct.c_void_p), ct.cast(rcv, ct.c_void_p), 4) == 0
            # ring: send 5 bytes to r+1, receive from r-1
            out = (ct.c_uint8 * 5)(*[100 + r] * 5)
            inn = (ct.c_uint8 * 5)()
            peer = (ct.c_int32 * 2)((r + 1) % P, (r - 1) % P)
            dirs = (ct.c_int32 * 2)(0, 1)
            bufs = (ct.c_void_p * 2)(ct.cast(out, ct.c_void_p), ct.cast(inn, ct.c_void_p))
            nb = (ct.c_int64 * 2)(5, 5)
            assert x.sendrecv(None, 2, peer, dirs, bufs, nb) == 0
            res[r] = (list(w), v[0], list(rcv), list(inn))
        except Exception as e:
            errs.append(e)
            g.bar.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for r in range(P):
        w, v, rcv, inn = res[r]
        assert w == [21, 0] and v == 6
        assert rcv == [0] * 4 + [1] * 4 + [2] * 4
        assert inn == [100 + (r - 1) % P] * 5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cplx, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from dist_model import sharded_gesvj_model
        tr = GlooTransport()
        # the raw callbacks first (as the library calls them)
        w = (ct.c_int64 * 1)(7 + rank)
        assert tr.xport.allreduce(None, ct.cast(w, ct.c_void_p), 1, 0) == 0 and w[0] == 7 + world - 1
        A = _case(cplx)
        res = sharded_gesvj_model(A, 16, tr, _rspec(cplx, A.shape[0]))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cplx", [False, True])
def test_gloo_world_size_2_bitwise(cplx):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cplx, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=600) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res = outs[0][1]
    assert np.array_equal(_bits(outs[1][1]["sigma"]), _bits(res["sigma"]))
    assert np.array_equal(outs[1][1]["perm"], res["perm"])
    assert list(local_columns(32, 16, 1, 2)) == list(outs[1][1]["cols"])
    _check_against_oracle(_case(cplx), cplx, [(o["cols"], o["U"], o["V"]) for _, o in outs], res)
