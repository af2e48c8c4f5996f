"""Out-of-bounds guards (compute-sanitizer is not available on the GPU pool):
every output is a slice in the middle of a larger buffer whose margins hold a
sentinel pattern; after the call the margins must be untouched.  Ragged sizes
put the kernels' tail paths at the slice edges."""
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

PAD = 4096  # elements of margin on each side
SENT = float.fromhex("0x1.dead0beefp+77")


@pytest.fixture(scope="module")
def J():
    import paper_2202_08361_b200 as J
    assert torch.cuda.is_available()
    return J


def _isfp(dtype):
    return dtype.is_floating_point or dtype.is_complex


def _guarded(n, dtype=torch.float64):
    buf = torch.full((n + 2 * PAD,), SENT if _isfp(dtype) else -12345, dtype=dtype, device="cuda")
    return buf, buf[PAD:PAD + n]


def _margins_intact(buf):
    m = torch.cat([buf[:PAD], buf[-PAD:]])
    ref = SENT if _isfp(buf.dtype) else -12345
    return bool((m == ref).all().item())


@pytest.mark.parametrize("f32", [False, True])
@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("r", [1, 31, 33, 511, 513, 4099])
def test_evd_outputs_stay_in_bounds(J, f32, cplx, r):
    dt = torch.float32 if f32 else torch.float64
    gen = (synth.evd_cfg2_f32 if cplx else synth.evd_cfg1_f32) if f32 else \
        (synth.evd_cfg2 if cplx else synth.evd_cfg1)
    ins = [torch.from_numpy(x).cuda() for x in gen(r)]
    bufs, out = {}, {}
    for k in ("lam1", "lam2", "cos", "sin_re") + (("sin_im",) if cplx else ()):
        bufs[k], out[k] = _guarded(r, dt)
    if not cplx:
        out["sin_im"] = None
    bufs["zeta"], out["zeta"] = _guarded(r, torch.int32)
    bufs["perm"], out["perm"] = _guarded((r + 31) // 32, torch.int32)
    J.evd2_batched(*ins, out=out)
    torch.cuda.synchronize()
    for k, b in bufs.items():
        assert _margins_intact(b), k


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("m", [1, 33, 257, 1025])
def test_norm_ef_outputs_stay_in_bounds(J, cplx, m):
    n = 13
    dt = torch.complex128 if cplx else torch.float64
    G = torch.randn(n, m + 3, dtype=dt, device="cuda").T[:m, :]  # ld = m + 3
    be, ce = _guarded(n)
    bf, cf = _guarded(n)
    b2, e2 = _guarded(n)
    b3, f2 = _guarded(n)
    J.norm_ef(G, col_e=ce, col_f=cf, col_e2=e2, col_f2=f2)
    torch.cuda.synchronize()
    assert all(_margins_intact(b) for b in (be, bf, b2, b3))


@pytest.mark.parametrize("m", [7, 1025, 3000])
def test_dgsscl_touches_only_q_columns(J, m):
    n, ld = 12, m + 5
    base = torch.randn(n * ld, dtype=torch.float64, device="cuda")
    G = base.view(n, ld).T[:m, :]
    pairs = torch.tensor([[0, 7], [3, 4], [10, 2]], dtype=torch.int32, device="cuda")
    ce, cf = J.colnorms(G)
    before = base.clone()
    J.dgsscl(G, pairs, ce, cf, torch.tensor([0.3, -0.2, 0.9], dtype=torch.float64, device="cuda"))
    torch.cuda.synchronize()
    changed = (base != before).view(n, ld)
    # only rows < m of the q columns (7, 4, 2) may change; padding rows never
    assert not changed[:, m:].any()
    for j in range(n):
        if j not in (7, 4, 2):
            assert not changed[j].any(), j


@pytest.mark.parametrize("cplx", [False, True])
def test_sweep_step_touches_only_its_pairs(J, cplx):
    m, n, ld = 1000, 16, 1003
    dt = torch.complex128 if cplx else torch.float64
    base = torch.randn(n * ld, dtype=dt, device="cuda") * 2.0 ** 900
    G = base.view(n, ld).T[:m, :]
    vbase = torch.eye(n, dtype=dt, device="cuda").T.contiguous()
    V = vbase.T
    pairs = torch.tensor([[0, 9], [4, 5]], dtype=torch.int32, device="cuda")
    before = base.clone()
    J.sweep_step(G, V, pairs)
    torch.cuda.synchronize()
    changed = (base != before).view(n, ld)
    assert not changed[:, m:].any()
    for j in range(n):
        if j not in (0, 9, 4, 5):
            assert not changed[j].any(), j


@pytest.mark.parametrize("cplx", [False, True])
def test_gesvj_batched_stays_in_its_matrices(J, cplx):
    b, m, n = 5, 64, 32
    dt = torch.complex128 if cplx else torch.float64
    sa, sv = m * n + 17, n * n + 9  # strides with gaps between the matrices
    abuf = torch.full((b * sa + 2 * PAD,), SENT, dtype=dt, device="cuda")
    vbuf = torch.full((b * sv + 2 * PAD,), SENT, dtype=dt, device="cuda")
    A = torch.as_strided(abuf[PAD:], (b, m, n), (sa, 1, m))
    A.copy_(torch.randn(b, n, m, dtype=dt, device="cuda").transpose(1, 2))
    V = torch.as_strided(vbuf[PAD:], (b, n, n), (sv, 1, n))
    sbuf, sig = _guarded(b * n)
    J.gesvj_batched(A, V=V, sigma=sig.view(b, n))
    torch.cuda.synchronize()
    assert _margins_intact(abuf) and _margins_intact(vbuf) and _margins_intact(sbuf)
    for k in range(b):  # the gaps between matrices
        assert bool((abuf[PAD + k * sa + m * n:PAD + (k + 1) * sa] == SENT).all().item())
        assert bool((vbuf[PAD + k * sv + n * n:PAD + (k + 1) * sv] == SENT).all().item())


@pytest.mark.parametrize("cplx", [False, True])
def test_gesvj_stays_in_its_arrays(J, cplx):
    m, n, ld = 300, 24, 307
    dt = torch.complex128 if cplx else torch.float64
    abuf = torch.full((n * ld + 2 * PAD,), SENT, dtype=dt, device="cuda")
    A = torch.as_strided(abuf[PAD:], (m, n), (1, ld))
    A.copy_(torch.randn(n, m, dtype=dt, device="cuda").T)
    vbuf = torch.full((n * (n + 3) + 2 * PAD,), SENT, dtype=dt, device="cuda")
    V = torch.as_strided(vbuf[PAD:], (n, n), (1, n + 3))
    res = J.gesvj(A, V=V, max_sweeps=30)
    torch.cuda.synchronize()
    assert res["status"] == 0
    assert _margins_intact(abuf) and _margins_intact(vbuf)
    pad_rows = abuf[PAD:PAD + n * ld].view(n, ld)[:, m:]
    assert bool((pad_rows == SENT).all().item())
    assert bool((vbuf[PAD:PAD + n * (n + 3)].view(n, n + 3)[:, n:] == SENT).all().item())


@pytest.mark.parametrize("cplx", [False, True])
def test_host_pipeline_stays_in_host_arrays(J, cplx):
    r = 5000
    arrs = synth.evd_cfg2(r) if cplx else synth.evd_cfg1(r)
    ins = [torch.from_numpy(a).pin_memory() for a in arrs] + ([] if cplx else [None])
    bufs, out = {}, {}
    for k in ("lam1", "lam2", "cos", "sin_re") + (("sin_im",) if cplx else ()):
        b = torch.full((r + 2 * PAD,), SENT, dtype=torch.float64).pin_memory()
        bufs[k], out[k] = b, b[PAD:PAD + r]
    if not cplx:
        out["sin_im"] = None
    for k, n_ in (("zeta", r), ("perm", (r + 31) // 32)):
        b = torch.full((n_ + 2 * PAD,), -12345, dtype=torch.int32).pin_memory()
        bufs[k], out[k] = b, b[PAD:PAD + n_]
    J.evd2_batched_host(*ins, out=out, chunk=1024)
    torch.cuda.synchronize()
    for k, b in bufs.items():
        ref = -12345 if k in ("zeta", "perm") else SENT
        assert bool((b[:PAD] == ref).all()) and bool((b[-PAD:] == ref).all()), k
