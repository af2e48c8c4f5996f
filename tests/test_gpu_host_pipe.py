"""GPU parity of the HOST-buffer entry points (jsvd_evd2_batched_host,
jsvd_gesvj_batched_host; include/jsvd.h) against the oracle, BITWISE, with
ragged chunkings that put chunk boundaries inside perm words' batches, make the
tail chunk short, and cycle every one of the three pipeline slots several times."""
import numpy as np
import pytest
import torch

import oracle as O
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def J():
    import paper_2202_08361_b200 as J
    assert torch.cuda.is_available()
    return J


def _host_out(J, r, dt, cplx, pinned):
    out = {k: torch.full((r,), 7.0, dtype=dt, pin_memory=pinned)
           for k in ("lam1", "lam2", "cos", "sin_re")}
    out["sin_im"] = torch.full((r,), 7.0, dtype=dt, pin_memory=pinned) if cplx else None
    out["zeta"] = torch.full((r,), 7, dtype=torch.int32, pin_memory=pinned)
    out["perm"] = torch.full(((r + 31) // 32,), 7, dtype=torch.int32, pin_memory=pinned)
    return out


def _bits(t):
    if t.is_complex():
        t = torch.view_as_real(t)
    return np.ascontiguousarray(t.numpy()).view(np.uint64)


def _compare(out, ref, cplx, f32):
    u = np.uint32 if f32 else np.uint64
    for k in ["lam1", "lam2", "cos", "sin_re"] + (["sin_im"] if cplx else []):
        a, b = out[k].numpy().view(u), ref[k].view(u)
        bad = np.nonzero(a != b)[0]
        assert bad.size == 0, (k, bad[:5])
    assert np.array_equal(out["zeta"].numpy(), ref["zeta"])
    assert np.array_equal(out["perm"].numpy().view(np.uint32), ref["perm"].view(np.uint32))


@pytest.mark.parametrize("f32", [False, True])
@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("r,chunk,pinned", [(1, 32, True), (31, 64, True), (4097, 1024, True),
                                            (100003, 4096, True), (100003, 32768, False),
                                            (65536, 8192, True)])
def test_evd2_host_bitwise(J, f32, cplx, r, chunk, pinned):
    if f32:
        arrs = synth.evd_cfg2_f32(r, seed=300 + r) if cplx else synth.evd_cfg1_f32(r, seed=300 + r)
        ref = O.evd2_batched_f32(*arrs, flags=0)
        dt = torch.float32
    else:
        arrs = synth.evd_cfg2(r, seed=300 + r) if cplx else synth.evd_cfg1(r, seed=300 + r)
        ref = O.evd2_batched(*arrs, flags=0)
        dt = torch.float64
    ins = [torch.from_numpy(a).pin_memory() if pinned else torch.from_numpy(a) for a in arrs]
    if not cplx:
        ins.append(None)
    out = _host_out(J, r, dt, cplx, pinned)
    s = torch.cuda.Stream()
    J.evd2_batched_host(*ins, out=out, chunk=chunk, stream=s)
    s.synchronize()
    _compare(out, ref, cplx, f32)


def test_evd2_host_equals_device_path_at_config_size(J):
    # configs[1] size (2^24 complex): host pipeline == device entry point, bitwise
    r = 1 << 24
    arrs = synth.evd_cfg2(r)
    ins = [torch.from_numpy(a).pin_memory() for a in arrs]
    out = J.evd2_batched_host(*ins)
    torch.cuda.synchronize()
    dev = J.evd2_batched(*[t.cuda() for t in ins])
    torch.cuda.synchronize()
    for k in ("lam1", "lam2", "cos", "sin_re", "sin_im"):
        assert torch.equal(out[k].view(torch.int64), dev[k].cpu().view(torch.int64)), k
    assert torch.equal(out["zeta"], dev["zeta"].cpu())
    assert torch.equal(out["perm"], dev["perm"].cpu())


def test_evd2_host_rejects_bad_arguments(J):
    x = torch.zeros(64, dtype=torch.float64)
    with pytest.raises(J.JsvdError):
        J.evd2_batched_host(x, x, x, chunk=48)  # not a multiple of 32
    with pytest.raises(ValueError):
        J.evd2_batched_host(x.cuda(), x, x)  # device tensor
    with pytest.raises(ValueError):
        J.evd2_batched_host(x, x, x, work=torch.empty(16, dtype=torch.uint8, device="cuda"))


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("batch,chunk", [(1, 1), (11, 3), (64, 64), (100, 16)])
def test_gesvj_batched_host_bitwise(J, cplx, batch, chunk):
    m, n = (64, 32) if cplx else (40, 24)
    if cplx:
        A = synth.svd_cfg4(batch)
    else:
        A = np.real(synth.svd_cfg4(batch, m=m, n=n))
    A = A.copy()
    A[batch // 2] *= 2.0 ** 900  # a matrix that needs the downscaling of P:1071-1115
    if batch > 3:
        A[3] = 0.0  # ERANK next to converging neighbours
    W, c, offs = J.batched_rspec(cplx, m)
    ref = O.gesvj_batched(A, O.RSpec.make(W, c, offs), max_sweeps=30)
    h = torch.from_numpy(np.ascontiguousarray(np.transpose(A, (0, 2, 1)))).transpose(1, 2)
    h = h.transpose(1, 2).contiguous().pin_memory().transpose(1, 2)
    out = J.gesvj_batched_host(h, max_sweeps=30, chunk=chunk)
    torch.cuda.synchronize()
    assert np.array_equal(out["status"].numpy(), ref["status"])
    assert np.array_equal(out["sweeps"].numpy(), ref["sweeps"])
    ok = [k for k in range(batch) if ref["status"][k] >= 0]
    def nb(a):
        return np.ascontiguousarray(a).view(np.uint64)
    for k in ("U", "V", "sigma"):
        assert np.array_equal(nb(out[k].numpy()[ok]), nb(ref[k][ok])), k
    # A itself is not modified
    assert np.array_equal(h.numpy(), A)


def test_gesvj_batched_host_equals_device_path_config4(J):
    bsz = 65536
    A = synth.svd_cfg4(bsz)
    h = torch.from_numpy(np.ascontiguousarray(np.transpose(A, (0, 2, 1)))).pin_memory().transpose(1, 2)
    out = J.gesvj_batched_host(h, max_sweeps=30, chunk=8192)
    g = h.cuda()
    tr = torch.empty(bsz, dtype=torch.int64, device="cuda")
    dev = J.gesvj_batched(g, max_sweeps=30, transforms=tr)
    torch.cuda.synchronize()
    for k in ("U", "V", "sigma"):
        assert np.array_equal(_bits(out[k]), _bits(dev[k].cpu())), k
    assert torch.equal(out["transforms"], tr.cpu())


@pytest.mark.parametrize("cplx", [False, True])
def test_gesvj_host_equals_device_path(J, cplx):
    rng = np.random.default_rng(12 + cplx)
    m, n, lda = 300, 24, 305
    A = rng.standard_normal((m, n)) * 2.0 ** rng.integers(-30, 30, (1, n))
    if cplx:
        A = A + 1j * rng.standard_normal((m, n))
    buf = np.zeros((n, lda), dtype=A.dtype)
    buf[:, :m] = A.T
    h = torch.from_numpy(buf).pin_memory().T[:m, :]  # host, column-major, lda = 305
    out = J.gesvj_host(h, max_sweeps=30)
    dev = J.gesvj(torch.from_numpy(np.ascontiguousarray(A.T)).cuda().T, max_sweeps=30)
    torch.cuda.synchronize()
    assert out["status"] == dev["status"] and out["sweeps"] == dev["sweeps"]
    assert out["tps"] == dev["tps"]
    for k in ("U", "V", "sigma"):
        assert np.array_equal(_bits(out[k].T.contiguous() if k != "sigma" else out[k]),
                              _bits(dev[k].T.contiguous().cpu() if k != "sigma" else dev[k].cpu())), k
    assert np.array_equal(h.numpy(), A)  # the host input is not modified


def test_evd2_host_two_threads_two_streams(J):
    # the shared fork event must order each call after ITS caller's
    # stream.  Two host threads, each first writing its pinned inputs from the
    # device on its own stream (D2H queued just before the call), then calling
    # the host pipeline on that stream: a call ordered after the other
    # thread's stream would upload stale inputs.
    import threading
    r, chunk = 200003, 8192
    arrs = [synth.evd_cfg2(r, seed=900 + t) for t in range(2)]
    refs = [O.evd2_batched(*a, flags=0) for a in arrs]
    errs = []

    def run(t):
        try:
            s = torch.cuda.Stream()
            dev_in = [torch.from_numpy(a).cuda() for a in arrs[t]]
            torch.cuda.synchronize()
            for it in range(4):
                ins = [torch.full((r,), 3.0, dtype=torch.float64, pin_memory=True) for _ in range(4)]
                with torch.cuda.stream(s):
                    for h, d in zip(ins, dev_in):
                        h.copy_(d, non_blocking=True)
                out = _host_out(J, r, torch.float64, True, True)
                J.evd2_batched_host(*ins, out=out, chunk=chunk, stream=s)
                s.synchronize()
                _compare(out, refs[t], True, False)
        except Exception as e:  # surfaced in the main thread
            errs.append(e)

    th = [threading.Thread(target=run, args=(t,)) for t in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs, errs


def test_gesvj_batched_host_rejects_shapes_before_queueing(J):
    # shapes jsvd_gesvj_batched rejects are rejected up front
    # (nothing queued), by the workspace query and by the call itself
    import ctypes as ct
    L = J.lib()
    work = torch.empty(1 << 22, dtype=torch.uint8, device="cuda")
    for m, n in ((130, 32), (64, 66), (64, 31), (16, 32)):
        with pytest.raises(J.JsvdError):
            J.gesvj_batched_host_workspace(False, m, n, 2)
        A = torch.zeros(2 * m * n, dtype=torch.float64, pin_memory=True)
        U = torch.zeros(2 * m * n, dtype=torch.float64, pin_memory=True)
        V = torch.zeros(2 * n * n, dtype=torch.float64, pin_memory=True)
        sg = torch.zeros(2 * n, dtype=torch.float64, pin_memory=True)
        st = L.jsvd_gesvj_batched_host(J.R64, 2, m, n, ct.c_void_p(A.data_ptr()),
                                       ct.c_void_p(U.data_ptr()), ct.c_void_p(V.data_ptr()),
                                       ct.c_void_p(sg.data_ptr()), 30, None, None, None, 2,
                                       ct.c_void_p(work.data_ptr()), work.numel(), None)
        assert st == -1, (m, n, st)  # JSVD_EINVAL
