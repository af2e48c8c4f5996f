"""GPU parity of the Jacobi-SVD entry points against the oracle, BITWISE:
jsvd_strategy_pairs, jsvd_sweep_step (every kernel geometry: single CTA and
2/4/8-CTA clusters), jsvd_gesvj (U, V, sigma, (e,f), sweeps, T per sweep).
The oracle is given the reduction spec R of DESIGN.md R#15 for (dtype, m),
written out here (and checked against what the library reports)."""
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


# The step kernel's reduction spec R (R#15), written out per
# (dtype, m) rather than queried from the library under test: W = 256 CL lanes
# (CL CTAs of 256 threads), element i on lane i mod W, lanes combined by xor
# offsets 16..1 (warp), 128, 64, 32 (warps of the CTA), then W/2 .. 256 (the
# CTAs of the cluster).  W is the smallest power of two >= 256 with W * NR >= m
# (NR = 16 real / 8 complex rows per lane in registers); beyond W = 2048 the
# kernel holds 2 NR rows per lane (half in shared memory), so W * 2 NR >= m.
_W_TABLE = {
    (False, 1): 256, (False, 7): 256, (False, 64): 256, (False, 255): 256, (False, 256): 256,
    (False, 257): 256, (False, 300): 256, (False, 1000): 256, (False, 2049): 256,
    (False, 4096): 256, (False, 8191): 512, (False, 16384): 1024, (False, 20001): 2048,
    (False, 65536): 2048,
    (True, 1): 256, (True, 7): 256, (True, 64): 256, (True, 255): 256, (True, 256): 256,
    (True, 257): 256, (True, 300): 256, (True, 1000): 256, (True, 2048): 256, (True, 2049): 512,
    (True, 4096): 512, (True, 8191): 1024, (True, 16384): 2048, (True, 20001): 2048,
    (True, 32768): 2048,
}
_W_TABLE.update({(c, m): 256 for c in (False, True) for m in (2, 4, 6, 8, 16, 40, 100, 512, 600)})


def rspec(J, cplx, m):
    W = _W_TABLE[(cplx, m)]
    offs = [16, 8, 4, 2, 1, 128, 64, 32] + [W >> k for k in range(1, 16) if (W >> k) >= 256]
    assert J.step_rspec(cplx, m) == (W, 1, tuple(offs)), (cplx, m)  # the library agrees
    return O.RSpec.make(W, 1, offs)


def colmajor_gpu(A):
    t = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()  # (n, m) row-major == (m, n) col-major
    return t.T


def to_np(t):
    return t.T.contiguous().cpu().numpy().T


def bits_equal(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    if a.shape != b.shape:
        return False
    if np.iscomplexobj(a):
        a, b = a.view(np.float64), b.view(np.float64)
    return np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("n,B", [(2, 2), (8, 8), (8, 2), (16, 4), (64, 16), (1024, 1024),
                                 (1024, 16), (96, 6)])
def test_strategy_pairs_match_oracle(J, n, B):
    for k in range(n - 1):
        g = J.strategy_pairs(n, B, k).cpu().numpy()
        assert np.array_equal(g, O.strategy_pairs(n, B, k)), (n, B, k)


def _scaled_input(rng, m, n, cplx, specials=True):
    A = rng.standard_normal((m, n)) * 2.0 ** rng.integers(-40, 40, n)
    if cplx:
        A = A + 1j * rng.standard_normal((m, n)) * 2.0 ** rng.integers(-40, 40, n)
    if specials and n >= 6:
        A[:, 1] = 0.0                                 # zero column (R#19)
        A[: max(1, m // 3), 2] = 5e-324 * 3           # subnormal entries
        A[:, 3] *= 2.0 ** -1000                       # tiny column
        A[:, 4] *= 2.0 ** 600                         # huge relative range
    # the step's precondition: pre-scaled as jsvd_gesvj would (||G||max <= omega/(4m))
    mx = np.abs(A.view(np.float64) if cplx else A).max()
    s = O.Fm(cplx, m) - int(np.floor(np.log2(mx))) - 1
    return np.asfortranarray(np.ldexp(A.real, s) + (1j * np.ldexp(A.imag, s) if cplx else 0))


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("m", [1, 7, 64, 255, 256, 257, 1000, 2049, 4096, 8191, 16384, 20001, 32768])
def test_sweep_step_bitwise(J, cplx, m):
    if not cplx and m == 32768:
        m = 65536  # the real 8-CTA cluster geometry
    n = 12
    rng = np.random.default_rng(m + 7 * cplx)
    A = _scaled_input(rng, m, n, cplx)
    V = np.asfortranarray(np.eye(n, dtype=A.dtype) + 0.0)
    R = rspec(J, cplx, m)
    G_ref, V_ref = A.copy(order="F"), V.copy(order="F")
    g, v = colmajor_gpu(A), colmajor_gpu(V)
    for k in range(3):
        pairs = O.strategy_pairs(n, n, k)
        ref = O.step(G_ref, V_ref, pairs, R)
        out = J.sweep_step(g, v, torch.from_numpy(pairs.astype(np.int32)).cuda())
        torch.cuda.synchronize()
        assert bits_equal(to_np(g), G_ref), (m, k)
        assert bits_equal(to_np(v), V_ref), (m, k)
        assert bits_equal(out["col_e"].cpu().numpy(), ref["col_e"])
        assert bits_equal(out["col_f"].cpu().numpy(), ref["col_f"])
        assert int(out["t"].item()) == ref["t"]
        assert out["mmax"].item() == ref["mmax"]


def test_sweep_step_partial_pairs_and_no_V(J):
    m, n = 300, 10
    rng = np.random.default_rng(3)
    A = _scaled_input(rng, m, n, False, specials=False)
    R = rspec(J, False, m)
    pairs = np.array([[0, 9], [4, 2]], np.int32)  # p > q on purpose in the second pair? no: p<q
    pairs = np.array([[0, 9], [2, 4]], np.int32)
    G_ref = A.copy(order="F")
    ref = O.step(G_ref, None, pairs, R)
    g = colmajor_gpu(A)
    out = J.sweep_step(g, None, torch.from_numpy(pairs).cuda())
    torch.cuda.synchronize()
    assert bits_equal(to_np(g), G_ref)
    assert int(out["t"].item()) == ref["t"] == 2


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("m,n,B", [(8, 8, 8), (64, 32, 32), (100, 20, 20), (257, 16, 4),
                                   (512, 64, 16), (600, 40, 40)])
def test_gesvj_bitwise(J, cplx, m, n, B):
    rng = np.random.default_rng(m * n + cplx)
    A = rng.standard_normal((m, n)) * (2.0 ** -rng.integers(0, 30, n))
    if cplx:
        A = A + 1j * rng.standard_normal((m, n))
    R = rspec(J, cplx, m)
    ref = O.gesvj(A, R, B=B, max_sweeps=40)
    g = colmajor_gpu(np.asfortranarray(A))
    out = J.gesvj(g, nblocks=B, max_sweeps=40)
    assert out["status"] == ref["status"]
    assert out["sweeps"] == ref["sweeps"]
    assert list(out["tps"]) == list(ref["tps"])
    assert bits_equal(to_np(out["U"]), ref["U"])
    assert bits_equal(to_np(out["V"]), ref["V"])
    assert bits_equal(out["sigma"].cpu().numpy(), ref["sigma"])
    assert bits_equal(out["sigma_e"].cpu().numpy(), ref["sigma_e"])
    assert bits_equal(out["sigma_f"].cpu().numpy(), ref["sigma_f"])


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("max_sweeps", [0, 1, 2])
def test_gesvj_capped_run_is_G_and_sigma_prime(J, cplx, max_sweeps):
    # Alg 4.1 line 41 (R#25): C = S -> no finalize; A holds
    # G = U Sigma' (scaled by 2^s), sigma Sigma' in column order, perm identity
    rng = np.random.default_rng(5 + cplx)
    A = rng.standard_normal((64, 16)) + (1j * rng.standard_normal((64, 16)) if cplx else 0)
    R = rspec(J, cplx, 64)
    ref = O.gesvj(A, R, max_sweeps=max_sweeps)
    out = J.gesvj(colmajor_gpu(np.asfortranarray(A)), max_sweeps=max_sweeps)
    assert out["status"] == ref["status"] == 1  # ENOCONV
    assert out["sweeps"] == ref["sweeps"] == max_sweeps and out["scale"] == ref["scale"]
    assert list(out["tps"]) == list(ref["tps"])
    for k in ("U", "V"):
        assert bits_equal(to_np(out[k]), ref[k]), k
    for k in ("sigma", "sigma_e", "sigma_f"):
        assert bits_equal(out[k].cpu().numpy(), ref[k]), k
    assert np.array_equal(out["perm"].cpu().numpy(), np.arange(16))


def test_gesvj_errors(J):
    with pytest.raises(J.JsvdError):
        J.gesvj(colmajor_gpu(np.zeros((8, 4))))
    bad = np.ones((8, 4))
    bad[2, 2] = np.nan
    with pytest.raises(J.JsvdError):
        J.gesvj(colmajor_gpu(bad))
    with pytest.raises(J.JsvdError):  # s0_adjust that would overflow G1 (R#40)
        J.gesvj(colmajor_gpu(np.ones((8, 4))), s0_adjust=1024 - O.Fm(False, 8) + 1)


@pytest.mark.parametrize("cplx,adj_from_K", [(False, 0), (False, 1), (True, 0), (True, 1),
                                              (True, 3)])
def test_gesvj_rescale_fires_bitwise(J, cplx, adj_from_K):
    # R#40: s0_adjust = K + 1 - F(m) + d starts at floor(lg M~1) = K + d, so
    # the Eq. (skr) check fires at step 0 (d >= 1) or in mid-run when a
    # component reaches 2^(K+1) (d = 0) -- the M-tilde "track" shortcut
    # (pairs with max(e) > K - 1 tracked) is exercised right at the boundary.
    K = 1020 if cplx else 1022
    rng = np.random.default_rng(70 + cplx + 3 * adj_from_K)
    fired = 0
    for m, n in ((2, 2), (4, 4), (6, 4), (8, 8), (40, 24)):
        A = rng.standard_normal((m, n)) + (1j * rng.standard_normal((m, n)) if cplx else 0)
        adj = K + 1 - O.Fm(cplx, m) + adj_from_K
        R = O.RSpec.make(256, 1, [16, 8, 4, 2, 1, 128, 64, 32])  # R#15 for m <= 2048
        assert J.step_rspec(cplx, m) == (256, 1, (16, 8, 4, 2, 1, 128, 64, 32))
        ref = O.gesvj(A, R, max_sweeps=40, s0_adjust=adj)
        out = J.gesvj(colmajor_gpu(np.asfortranarray(A)), max_sweeps=40, s0_adjust=adj)
        assert out["status"] == ref["status"] and out["sweeps"] == ref["sweeps"]
        assert out["scale"] == ref["scale"], (m, n)
        assert bits_equal(to_np(out["U"]), ref["U"]) and bits_equal(to_np(out["V"]), ref["V"])
        for k in ("sigma", "sigma_e", "sigma_f"):
            assert bits_equal(out[k].cpu().numpy(), ref[k]), k
        base = O.gesvj(A, R, max_sweeps=40)
        fired += ref["scale"] < base["scale"] + adj
    # d >= 1: floor(lg M~1) = K + d fires at step 0 on every input; d = 0 fires
    # once a component reaches 2^(K+1) (on some of these inputs)
    assert fired >= (5 if adj_from_K else 1)


def test_config3_full_size_step_bitwise(J):
    # BASELINE configs[2] at full size (4096 x 1024): the first 3 steps of
    # jsvd_gesvj's first sweep, GPU vs oracle, after the same initial scaling.
    A, _ = synth.svd_cfg3()
    m, n = A.shape
    R = rspec(J, False, m)
    s0 = O.Fm(False, m) - int(np.floor(np.log2(np.abs(A).max()))) - 1
    G = np.asfortranarray(np.ldexp(A, s0))
    V = np.asfortranarray(np.eye(n))
    g, v = colmajor_gpu(G), colmajor_gpu(V)
    for k in range(3):
        pairs = O.strategy_pairs(n, n, k)
        ref = O.step(G, V, pairs, R)
        out = J.sweep_step(g, v, torch.from_numpy(pairs.astype(np.int32)).cuda())
        torch.cuda.synchronize()
        assert int(out["t"].item()) == ref["t"] == n // 2
        assert bits_equal(to_np(g), G) and bits_equal(to_np(v), V)


def test_config3_full_size_gesvj_two_sweeps_bitwise(J):
    # BASELINE configs[2] at full size through the driver the bench times
    # (jsvd_gesvj, flat round-robin, the same call as bench.py's gesvj_r64)
    # capped at two sweeps (2046 steps; the oracle takes seconds): status
    # ENOCONV, G = U Sigma', V, Sigma' in column order, T per sweep and the
    # final scale, all bitwise
    A, _ = synth.svd_cfg3()
    m, n = A.shape
    R = rspec(J, False, m)
    ref = O.gesvj(A, R, max_sweeps=2)
    out = J.gesvj(colmajor_gpu(np.asfortranarray(A)), max_sweeps=2)
    torch.cuda.synchronize()
    assert out["status"] == ref["status"] == 1 and out["sweeps"] == ref["sweeps"] == 2
    assert out["scale"] == ref["scale"] and list(out["tps"]) == list(ref["tps"])
    for k in ("U", "V"):
        assert bits_equal(to_np(out[k]), ref[k]), k
    for k in ("sigma", "sigma_e", "sigma_f"):
        assert bits_equal(out[k].cpu().numpy(), ref[k]), k


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("m,n", [(2, 2), (8, 6), (64, 32), (64, 16), (64, 30), (33, 32), (100, 40),
                                 (128, 64)])
def test_gesvj_batched_bitwise(J, cplx, m, n):
    rng = np.random.default_rng(m + n + cplx)
    b = 5
    A = rng.standard_normal((b, m, n)) * 2.0 ** rng.integers(-20, 20, (b, 1, n))
    if cplx:
        A = A + 1j * rng.standard_normal((b, m, n))
    A[1, :, 0] = 0.0  # a zero column
    W, c, offs = J.batched_rspec(cplx, m)
    ref = O.gesvj_batched(A, O.RSpec.make(W, c, offs), max_sweeps=40)
    g = torch.from_numpy(np.ascontiguousarray(np.transpose(A, (0, 2, 1)))).cuda().transpose(1, 2)
    out = J.gesvj_batched(g, max_sweeps=40)
    torch.cuda.synchronize()
    assert np.array_equal(out["status"].cpu().numpy(), ref["status"])
    assert np.array_equal(out["sweeps"].cpu().numpy(), ref["sweeps"])
    U = out["U"].transpose(1, 2).contiguous().cpu().numpy().transpose(0, 2, 1)
    V = out["V"].transpose(1, 2).contiguous().cpu().numpy().transpose(0, 2, 1)
    assert bits_equal(U, ref["U"]) and bits_equal(V, ref["V"])
    assert bits_equal(out["sigma"].cpu().numpy(), ref["sigma"])


def test_config4_batched_sampled_bitwise(J):
    # BASELINE configs[3] at full size in the bench's launch configuration
    # (65536 x 64 x 32 complex, one CTA per matrix); the oracle checks a
    # random sample of 64 matrices one by one.
    bsz, m, n = 65536, 64, 32
    A = synth.svd_cfg4(bsz)
    g = torch.from_numpy(np.ascontiguousarray(np.transpose(A, (0, 2, 1)))).cuda().transpose(1, 2)
    out = J.gesvj_batched(g, max_sweeps=30)
    torch.cuda.synchronize()
    assert (out["status"] == 0).all()
    idx = np.sort(np.random.default_rng(2).choice(bsz, 64, replace=False))
    W, c, offs = J.batched_rspec(True, m)
    ref = O.gesvj_batched(A[idx], O.RSpec.make(W, c, offs), max_sweeps=30)
    U = out["U"][idx].transpose(1, 2).contiguous().cpu().numpy().transpose(0, 2, 1)
    assert bits_equal(U, ref["U"])
    assert bits_equal(out["sigma"][idx].cpu().numpy(), ref["sigma"])
    # north_star tolerances on the GPU result: sigma vs LAPACK, residual, orthogonality
    s = np.linalg.svd(A[idx], compute_uv=False)
    assert (np.abs(out["sigma"][idx].cpu().numpy() - s) / s).max() <= 1e-12


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("max_sweeps", [2, 40])
def test_gesvj_batched_mixed_status_and_caps(J, cplx, max_sweeps):
    # matrices that stop at different sweeps share CTAs (two per CTA for n <= 32):
    # a zero matrix (ERANK), a non-finite one (ENONFINITE), an already
    # orthogonal one (1 sweep), capped runs (ENOCONV) next to converging ones
    rng = np.random.default_rng(90 + cplx + max_sweeps)
    b, m, n = 7, 40, 24
    A = rng.standard_normal((b, m, n)) * 2.0 ** rng.integers(-30, 30, (b, 1, n))
    if cplx:
        A = A + 1j * rng.standard_normal((b, m, n))
    A[2] = 0.0
    A[3, 5, 7] = np.nan
    Q, _ = np.linalg.qr(rng.standard_normal((m, n)))
    A[4] = Q * 2.0 ** np.arange(n)[None, :]  # orthogonal columns with distinct norms
    W, c, offs = J.batched_rspec(cplx, m)
    ref = O.gesvj_batched(A, O.RSpec.make(W, c, offs), max_sweeps=max_sweeps)
    g = torch.from_numpy(np.ascontiguousarray(np.transpose(A, (0, 2, 1)))).cuda().transpose(1, 2)
    out = J.gesvj_batched(g, max_sweeps=max_sweeps)
    torch.cuda.synchronize()
    assert np.array_equal(out["status"].cpu().numpy(), ref["status"])
    assert np.array_equal(out["sweeps"].cpu().numpy(), ref["sweeps"])
    ok = [k for k in range(b) if ref["status"][k] >= 0]
    U = out["U"].transpose(1, 2).contiguous().cpu().numpy().transpose(0, 2, 1)
    V = out["V"].transpose(1, 2).contiguous().cpu().numpy().transpose(0, 2, 1)
    assert bits_equal(U[ok], ref["U"][ok]) and bits_equal(V[ok], ref["V"][ok])
    assert bits_equal(out["sigma"].cpu().numpy()[ok], ref["sigma"][ok])


@pytest.mark.parametrize("cplx", [False, True])
def test_gesvj_batched_v_placement_is_invisible(J, monkeypatch, cplx):
    # half of the working V in shared memory (default) or all of it in A's
    # storage (JSVD_BATCHED_VH=0): the same arithmetic, so the same bits
    rng = np.random.default_rng(31 + cplx)
    b, m, n = 40, 64, 32
    A = rng.standard_normal((b, m, n)) * 2.0 ** rng.integers(-40, 40, (b, 1, n))
    if cplx:
        A = A + 1j * rng.standard_normal((b, m, n))
    outs = []
    for vh in ("1", "0"):
        monkeypatch.setenv("JSVD_BATCHED_VH", vh)
        g = torch.from_numpy(np.ascontiguousarray(np.transpose(A, (0, 2, 1)))).cuda().transpose(1, 2)
        o = J.gesvj_batched(g, max_sweeps=30)
        torch.cuda.synchronize()
        outs.append({k: o[k].transpose(1, 2).contiguous().cpu() if k in ("U", "V") else o[k].cpu()
                     for k in ("U", "V", "sigma", "sweeps", "status")})
    for k in outs[0]:
        a, c = outs[0][k], outs[1][k]
        if a.is_complex():
            a, c = torch.view_as_real(a), torch.view_as_real(c)
        assert torch.equal(a, c), k


@pytest.mark.parametrize("cplx", [False, True])
def test_gesvj_batched_rescale_and_cap_bitwise(J, cplx):
    # the batched kernel's own rescale (every step, flat RR) and its line-41
    # branch: s0_adjust = K + 1 - F(m) (fires in mid-run, R#40), and a 2-sweep
    # cap (ENOCONV: G = U Sigma', Sigma' unsorted, R#25); scale per matrix
    K = 1020 if cplx else 1022
    rng = np.random.default_rng(123 + cplx)
    for m, n in ((64, 32), (16, 16), (40, 24)):
        b = 9
        A = rng.standard_normal((b, m, n)) + (1j * rng.standard_normal((b, m, n)) if cplx else 0)
        W, c, offs = J.batched_rspec(cplx, m)
        assert (W, c, offs) == (8, 1, (4, 2, 1))  # R#15: 8 lanes per pair for m <= 64
        R = O.RSpec.make(8, 1, [4, 2, 1])
        for kw in (dict(s0_adjust=K + 1 - O.Fm(cplx, m)), dict(max_sweeps=2)):
            ref = O.gesvj_batched(A, R, **{"max_sweeps": 40, **kw})
            g = torch.from_numpy(np.ascontiguousarray(np.transpose(A, (0, 2, 1)))).cuda().transpose(1, 2)
            sc = torch.empty(b, dtype=torch.int32, device="cuda")
            out = J.gesvj_batched(g, scale=sc, **{"max_sweeps": 40, **kw})
            torch.cuda.synchronize()
            assert np.array_equal(out["status"].cpu().numpy(), ref["status"]), kw
            assert np.array_equal(out["sweeps"].cpu().numpy(), ref["sweeps"]), kw
            assert np.array_equal(sc.cpu().numpy(), ref["scale"]), kw
            U = out["U"].transpose(1, 2).contiguous().cpu().numpy().transpose(0, 2, 1)
            V = out["V"].transpose(1, 2).contiguous().cpu().numpy().transpose(0, 2, 1)
            assert bits_equal(U, ref["U"]) and bits_equal(V, ref["V"]), kw
            assert bits_equal(out["sigma"].cpu().numpy(), ref["sigma"]), kw


# ------------------------------------------- the paths configs[4] takes (R#15)
@pytest.mark.parametrize("cplx,m,nv", [(True, 32768, 8192), (True, 16384, 8192),
                                       (True, 2048, 1024), (True, 2048, 1030),
                                       (False, 4096, 1024), (False, 65536, 8192),
                                       (True, 300, 1500)])
def test_sweep_step_long_V_bitwise(J, cplx, m, nv):
    # Alg 3.4 applied to V with l = n rows: V has nv rows (the
    # order of the whole SVD) while the step holds 8 columns (4 pairs), as a
    # column-block rank does.  nv > 2 W reaches the V rows of cluster ranks
    # >= 1 and the strided tail loop of the step kernel; complex m <= 2048 is
    # the single-CTA (W = 256) geometry with a tail beyond row 512.
    ncols = 8
    rng = np.random.default_rng(m + nv + cplx)
    A = _scaled_input(rng, m, ncols, cplx, specials=False)
    V = rng.standard_normal((nv, ncols)) + (1j * rng.standard_normal((nv, ncols)) if cplx else 0)
    V = np.asfortranarray(V)
    R = rspec(J, cplx, m)
    G_ref, V_ref = A.copy(order="F"), V.copy(order="F")
    g, v = colmajor_gpu(A), colmajor_gpu(V)
    for k in range(2):
        pairs = np.array([[0, 5], [1, 7], [2, 4], [3, 6]] if k == 0 else [[0, 1], [2, 3], [4, 5], [6, 7]],
                         np.int32)
        ref = O.step(G_ref, V_ref, pairs, R)
        out = J.sweep_step(g, v, torch.from_numpy(pairs).cuda())
        torch.cuda.synchronize()
        assert int(out["t"].item()) == ref["t"] == 4
        assert bits_equal(to_np(g), G_ref), k
        assert bits_equal(to_np(v), V_ref), k
        assert out["mmax"].item() == ref["mmax"]


@pytest.mark.parametrize("pf", ["0", "3"])
def test_sweep_step_l2_prefetch_is_invisible(J, monkeypatch, pf):
    # the long-column step's bulk L2 prefetch of the pair pf pairs ahead (its
    # G columns and V columns) is a hint: 12 pairs of complex 32768-row
    # columns, with and without it, bitwise against the oracle
    monkeypatch.setenv("JSVD_STEP_PF", pf)
    cplx, m, ncols = True, 32768, 24
    rng = np.random.default_rng(29)
    A = _scaled_input(rng, m, ncols, cplx, specials=False)
    V = np.asfortranarray(np.eye(ncols) + 0j)
    R = rspec(J, cplx, m)
    G_ref, V_ref = A.copy(order="F"), V.copy(order="F")
    g, v = colmajor_gpu(A), colmajor_gpu(V)
    pairs = O.strategy_pairs(ncols, ncols, 0).astype(np.int32)
    ref = O.step(G_ref, V_ref, pairs, R)
    out = J.sweep_step(g, v, torch.from_numpy(pairs).cuda())
    torch.cuda.synchronize()
    assert int(out["t"].item()) == ref["t"]
    assert bits_equal(to_np(g), G_ref) and bits_equal(to_np(v), V_ref)


def test_config5_full_size_step_sampled_bitwise(J):
    # BASELINE configs[4] at full size (complex 32768 x 8192, 4.3 GB) in the
    # bench's launch configuration: one step of all 4096 pairs (block RR,
    # B = 16) of the scaled matrix with V = I of order 8192; the oracle
    # recomputes 6 sampled pairs from their columns before the step.
    m, n = 32768, 8192
    g, _ = synth.svd_cfg5_torch(m, n, device="cuda")  # (m, n) column-major complex128
    mx = torch.view_as_real(g).abs().max().item()
    s0 = O.Fm(True, m) - int(np.floor(np.log2(mx))) - 1
    torch.view_as_real(g).mul_(2.0 ** s0)  # exact power-of-two scaling (no subnormals here)
    v = torch.eye(n, dtype=torch.complex128, device="cuda").T.contiguous().T
    step = 600  # a phase-II step of the block ordering
    pairs = J.strategy_pairs(n, 16, step)
    sample = np.random.default_rng(1).choice(n // 2, 6, replace=False)
    pl = pairs.cpu().numpy()[sample]
    cols = pl.reshape(-1)
    G0 = np.asfortranarray(g[:, cols].cpu().numpy())
    V0 = np.asfortranarray(v[:, cols].cpu().numpy())
    out = J.sweep_step(g, v, pairs)
    torch.cuda.synchronize()
    local = np.arange(12, dtype=np.int32).reshape(6, 2)
    ref = O.step(G0, V0, local, rspec(J, True, m))
    assert bits_equal(g[:, cols].cpu().numpy(), G0)
    assert bits_equal(v[:, cols].cpu().numpy(), V0)
    ce, cf = out["col_e"].cpu().numpy(), out["col_f"].cpu().numpy()
    assert bits_equal(ce[cols], ref["col_e"]) and bits_equal(cf[cols], ref["col_f"])


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("kind", ["gauss", "graded", "tiny_entries", "zeros", "rank_def", "rescale"])
def test_gesvj_batched_fast_mode_is_invisible(J, monkeypatch, cplx, kind):
    # the batched kernel keeps G~ = G 2^-cs in shared memory
    # while every value is 0 or in [2^-400, 2^16]; the fast and the exact mode
    # (JSVD_BATCHED_FAST=0) give the same bits, and both equal the oracle --
    # including inputs that start outside the fast mode, leave it in mid-run
    # (cancellation to tiny values, tiny C / S), or rescale (R#40).
    rng = np.random.default_rng(55 + cplx)
    b, m, n = 24, 64, 32
    A = rng.standard_normal((b, m, n)) + (1j * rng.standard_normal((b, m, n)) if cplx else 0)
    adj = 0
    if kind == "graded":
        A = A * 2.0 ** rng.integers(-180, 180, (b, 1, n))
    elif kind == "tiny_entries":
        A[:, ::7, ::5] *= 2.0 ** -450          # beyond the fast range from the start
        A[::3, 5, 9] = 5e-324                   # subnormal entries
    elif kind == "zeros":
        A[:, 3, :] = 0.0
        A[::2, :, 4] = 0.0
    elif kind == "rank_def":
        A[:, :, 7] = A[:, :, 3] * 2.0 ** 9     # parallel columns: cancellation to ~0
        A[:, :, 11] = A[:, :, 2] + 2.0 ** -420 * A[:, :, 5]
    elif kind == "rescale":
        adj = (1021 if cplx else 1023) - O.Fm(cplx, m)
    R = O.RSpec.make(8, 1, [4, 2, 1])
    ref = O.gesvj_batched(A, R, max_sweeps=40, s0_adjust=adj)
    outs = []
    for fast in ("1", "0"):
        monkeypatch.setenv("JSVD_BATCHED_FAST", fast)
        g = torch.from_numpy(np.ascontiguousarray(np.transpose(A, (0, 2, 1)))).cuda().transpose(1, 2)
        sc = torch.empty(b, dtype=torch.int32, device="cuda")
        o = J.gesvj_batched(g, max_sweeps=40, scale=sc, s0_adjust=adj)
        torch.cuda.synchronize()
        outs.append(o)
        assert np.array_equal(o["status"].cpu().numpy(), ref["status"]), fast
        assert np.array_equal(o["sweeps"].cpu().numpy(), ref["sweeps"]), fast
        assert np.array_equal(sc.cpu().numpy(), ref["scale"]), fast
        ok = [k for k in range(b) if ref["status"][k] >= 0]
        U = o["U"].transpose(1, 2).contiguous().cpu().numpy().transpose(0, 2, 1)
        V = o["V"].transpose(1, 2).contiguous().cpu().numpy().transpose(0, 2, 1)
        assert bits_equal(U[ok], ref["U"][ok]) and bits_equal(V[ok], ref["V"][ok]), fast
        assert bits_equal(o["sigma"].cpu().numpy()[ok], ref["sigma"][ok]), fast


@pytest.mark.parametrize("fast", ["0", "1"])
@pytest.mark.parametrize("cplx", [False, True])
def test_step_both_paths_bitwise(J, monkeypatch, fast, cplx):
    # the step kernel's scaled single-pass norms + dot and its
    # exact three-round path (JSVD_STEP_FAST=0) give the oracle's bits: sweep
    # steps with zero, subnormal, tiny (2^-1000) and huge (2^600) columns at
    # the cluster geometries, and full SVDs with block ordering whose scale
    # sits at the top of the range (s0_adjust: floor(lg M~) = K, then K + 1)
    monkeypatch.setenv("JSVD_STEP_FAST", fast)
    for m in (300, 4096 if not cplx else 2049, 20001):
        n = 12
        rng = np.random.default_rng(m + 3 * cplx + 11)
        A = _scaled_input(rng, m, n, cplx)
        V = np.asfortranarray(np.eye(n, dtype=A.dtype) + 0.0)
        R = rspec(J, cplx, m)
        G_ref, V_ref = A.copy(order="F"), V.copy(order="F")
        g, v = colmajor_gpu(A), colmajor_gpu(V)
        for k in range(3):
            pairs = O.strategy_pairs(n, n, k)
            ref = O.step(G_ref, V_ref, pairs, R)
            out = J.sweep_step(g, v, torch.from_numpy(pairs.astype(np.int32)).cuda())
            torch.cuda.synchronize()
            assert bits_equal(to_np(g), G_ref) and bits_equal(to_np(v), V_ref), (m, k)
            assert bits_equal(out["col_e"].cpu().numpy(), ref["col_e"]), (m, k)
            assert bits_equal(out["col_f"].cpu().numpy(), ref["col_f"]), (m, k)
    K = 1020 if cplx else 1022
    m, n = 96, 64
    rng = np.random.default_rng(5 + cplx)
    A = rng.standard_normal((m, n)) + (1j * rng.standard_normal((m, n)) if cplx else 0)
    R = O.RSpec.make(256, 1, [16, 8, 4, 2, 1, 128, 64, 32])
    for adj in (0, K + 1 - O.Fm(cplx, m)):
        ref = O.gesvj(A, R, B=16, max_sweeps=30, s0_adjust=adj)
        out = J.gesvj(colmajor_gpu(np.asfortranarray(A)), nblocks=16, max_sweeps=30, s0_adjust=adj)
        assert list(out["tps"]) == list(ref["tps"]) and out["scale"] == ref["scale"], adj
        assert bits_equal(to_np(out["U"]), ref["U"]) and bits_equal(to_np(out["V"]), ref["V"]), adj
        assert bits_equal(out["sigma"].cpu().numpy(), ref["sigma"]), adj
