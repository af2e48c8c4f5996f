"""GPU parity of jsvd_evd2_batched_f32 (the single-precision EVD)
against the binary32 oracle: BITWISE on every output stream (lambda1, lambda2,
cos, sin, zeta, perm words).  Calls go through the C ABI (libjsvd.so)."""
import numpy as np
import pytest
import torch

import oracle as O
import synth

pytestmark = pytest.mark.gpu

FMAX = float(np.finfo(np.float32).max)
MU = float(np.finfo(np.float32).smallest_subnormal)


@pytest.fixture(scope="module")
def J():
    import paper_2202_08361_b200 as J
    assert torch.cuda.is_available()
    return J


def _run(J, arrs, flags, offset=0):
    """offset=1 shifts every stream by one element -> 4-byte-aligned scalar path."""
    g = []
    for a in arrs:
        t = torch.empty(a.size + offset, dtype=torch.float32, device="cuda")
        t[offset:].copy_(torch.from_numpy(a))
        g.append(t[offset:])
    r = arrs[0].size
    out = None
    if offset:
        out = {k: torch.empty(r + 1, dtype=torch.float32, device="cuda")[1:]
               for k in ("lam1", "lam2", "cos", "sin_re", "sin_im")}
        if len(arrs) == 3:
            out["sin_im"] = None
        out["zeta"] = torch.empty(r, dtype=torch.int32, device="cuda")
        out["perm"] = torch.empty((r + 31) // 32, dtype=torch.int32, device="cuda")
    res = J.evd2_batched(*g, flags=flags, out=out)
    torch.cuda.synchronize()
    return {k: (v.cpu().numpy() if v is not None else None) for k, v in res.items()}


def _compare(gpu, ref, cplx):
    for k in ["lam1", "lam2", "cos", "sin_re"] + (["sin_im"] if cplx else []):
        a, b = gpu[k].view(np.uint32), ref[k].view(np.uint32)
        bad = np.nonzero(a != b)[0]
        assert bad.size == 0, (k, bad[:5], gpu[k][bad[:5]], ref[k][bad[:5]])
    assert np.array_equal(gpu["zeta"], ref["zeta"])
    assert np.array_equal(gpu["perm"].view(np.uint32), ref["perm"])


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("flags", [0, 1, 2, 3])
@pytest.mark.parametrize("r", [1, 3, 4, 5, 31, 33, 127, 128, 129, 1023, 1024, 1025, 4099])
def test_ragged_sizes_all_flags_f32(J, cplx, flags, r):
    arrs = synth.evd_cfg2_f32(r, seed=200 + r) if cplx else synth.evd_cfg1_f32(r, seed=200 + r)
    ref = O.evd2_batched_f32(*arrs, flags=flags)
    _compare(_run(J, arrs, flags), ref, cplx)
    _compare(_run(J, arrs, flags, offset=1), ref, cplx)


def _specials():
    vals = [0.0, -0.0, MU, -MU, 2.0 ** -126, -(2.0 ** -126), MU * 3, 1.0, -1.0, FMAX, -FMAX,
            FMAX / 8, 2.0 ** 124, 1.5 * 2.0 ** 127, 0.5, 3.0, 1e-30, 1e30]
    rng = np.random.default_rng(0)
    rows = [rng.choice(vals, 4) for _ in range(20000)]
    rows += [[FMAX / 8, FMAX / 8, MU, s * MU] for s in (1, -1)]  # Eq. (5.1) analogue
    rows += [[0.0, 0.0, 0.0, 0.0], [-0.0, 0.0, -0.0, 0.0], [0.0, 0.0, MU, 0.0]]
    A = np.array(rows, dtype=np.float32)
    return tuple(np.ascontiguousarray(A[:, k]) for k in range(4))


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("flags", [0, 3])
def test_special_values_bitwise_f32(J, cplx, flags):
    arrs = _specials()
    if not cplx:
        arrs = arrs[:3]
    _compare(_run(J, arrs, flags), O.evd2_batched_f32(*arrs, flags=flags), cplx)


@pytest.mark.parametrize("cplx", [False, True])
def test_config_size_bitwise_f32(J, cplx):
    # the single-precision analogues of configs[0] (2^20) and configs[1] (2^24 here)
    arrs = synth.evd_cfg2_f32(1 << 24) if cplx else synth.evd_cfg1_f32(1 << 20)
    _compare(_run(J, arrs, 0), O.evd2_batched_f32(*arrs), cplx)


def test_f32_rejects_mixed_dtypes(J):
    x = torch.zeros(8, dtype=torch.float32, device="cuda")
    y = torch.zeros(8, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        J.evd2_batched(x, x, y)
