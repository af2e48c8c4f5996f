"""The column-block-sharded SVD (paper_2202_08361_b200.dist) on CPU:
schedule properties against the oracle's block round-robin, and an end-to-end
world_size-2 gloo run (oracle compute) that must be BITWISE identical to the
oracle's single-process SVD with the same ordering (nblocks = 16)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2202_08361_b200.dist import (BlockSchedule, LocalRanks, TorchDistRanks, gather_columns,
                                        gesvj_dist, scatter_columns)


@pytest.mark.parametrize("n", [32, 64, 96, 128])
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_schedule_matches_oracle_block_round_robin(n, P):
    S = BlockSchedule(n, 16, P)
    for k in range(n - 1):
        got = np.concatenate([S.global_pairs(r, k) for r in range(P)])
        ref = O.strategy_pairs(n, 16, k)
        assert sorted(map(tuple, got.tolist())) == sorted(map(tuple, ref.tolist())), (k,)
        for r in range(P):
            loc = S.local_pairs(r, k).reshape(-1)
            assert len(set(loc.tolist())) == loc.size and loc.max() < S.nslots * S.b
        assert S.is_checkpoint(k) == O.strategy_is_checkpoint(n, 16, k)


def test_moves_rotate_the_circle_back_after_a_sweep():
    for P in (1, 2, 4, 8):
        S = BlockSchedule(64, 16, P)
        hold = {(r, s): S.local_block(r, s, 0) for r in range(P) for s in range(S.nslots)}
        for rnd in range(15):
            new = {}
            for sr, ss, dr, ds in S.moves():
                new[(dr, ds)] = hold[(sr, ss)]
            new[S.owner(0)] = hold[S.owner(0)]
            hold = new
            assert all(hold[(r, s)] == S.local_block(r, s, rnd + 1)
                       for r in range(P) for s in range(S.nslots))
        assert all(hold[(r, s)] == S.local_block(r, s, 0) for r in range(P) for s in range(S.nslots))
        # at most two blocks leave and two arrive per rank and round
        sent = {}
        for sr, ss, dr, ds in S.moves():
            if sr != dr:
                sent[sr] = sent.get(sr, 0) + 1
        assert max(sent.values(), default=0) <= 2


def _case(cplx, m=64, n=32, seed=5):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, n)) * 2.0 ** rng.integers(-10, 10, n)
    if cplx:
        A = A + 1j * rng.standard_normal((m, n))
    return A


def _rspec(cplx, m):
    import paper_2202_08361_b200 as J  # host-only query, no GPU needed
    return O.RSpec.make(*J.step_rspec(cplx, m))


def _check_against_oracle(A, cplx, out_parts, sched, res):
    R = _rspec(cplx, A.shape[0])
    ref = O.gesvj(A, R, B=16, max_sweeps=30)
    U = np.array(gather_columns([p[0] for p in out_parts], sched)).T
    V = np.array(gather_columns([p[1] for p in out_parts], sched)).T
    perm = res["perm"]
    assert res["sweeps"] == ref["sweeps"] and res["status"] == ref["status"]
    assert list(res["tps"]) == list(ref["tps"])
    for got, exp in ((U[:, perm], ref["U"]), (V[:, perm], ref["V"]),
                     (res["sigma"], ref["sigma"]), (res["sigma_e"], ref["sigma_e"]),
                     (res["sigma_f"], ref["sigma_f"])):
        g, e = np.ascontiguousarray(got), np.ascontiguousarray(exp)
        if np.iscomplexobj(g):
            g, e = g.view(np.float64), e.view(np.float64)
        assert np.array_equal(g.view(np.uint64), e.view(np.uint64))


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("P", [1, 2, 4])
def test_virtual_ranks_oracle_compute_bitwise(cplx, P):
    from dist_oracle_compute import OracleCompute
    A = _case(cplx)
    m, n = A.shape
    S = BlockSchedule(n, 16, P)
    dt = torch.complex128 if cplx else torch.float64
    Gts = [torch.from_numpy(np.ascontiguousarray(A[:, scatter_columns(None, S, r)].T)).to(dt)
           for r in range(P)]
    res = gesvj_dist(Gts, S, LocalRanks(P), OracleCompute(_rspec(cplx, m)), cplx=cplx)
    parts = [(res["Gts"][r].numpy(), res["Vts"][r].numpy()) for r in range(P)]
    _check_against_oracle(A, cplx, parts, S, res)


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
        from dist_oracle_compute import OracleCompute
        A = _case(cplx)
        m, n = A.shape
        S = BlockSchedule(n, 16, world)
        dt = torch.complex128 if cplx else torch.float64
        G = torch.from_numpy(np.ascontiguousarray(A[:, scatter_columns(None, S, rank)].T)).to(dt)
        res = gesvj_dist([G], S, TorchDistRanks(), OracleCompute(_rspec(cplx, m)), cplx=cplx)
        q.put((rank, res["Gts"][0].numpy(), res["Vts"][0].numpy(),
               {k: res[k] for k in ("sigma", "sigma_e", "sigma_f", "perm", "sweeps", "tps", "status")}))
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
    A = _case(cplx)
    S = BlockSchedule(A.shape[1], 16, 2)
    res = outs[0][3]
    for o in outs[1:]:  # every rank agrees on sigma / perm / sweeps
        assert np.array_equal(o[3]["sigma"], res["sigma"]) and np.array_equal(o[3]["perm"], res["perm"])
    _check_against_oracle(A, cplx, [(o[1], o[2]) for o in outs], S, res)
