"""ctypes marshalling for oracle/liboracle.so (TEST INFRASTRUCTURE ONLY).

No arithmetic of the method lives here: every function converts numpy arrays
to pointers and calls the C oracle (oracle/jsvd_oracle.c).
"""
import ctypes as ct
import os

import numpy as np

from .build import LIB, build

__all__ = [
    "RSpec", "lib", "hypot", "zeta", "evd2_one", "evd2_batched", "colnorm", "dot", "cvg",
    "hypot_f32", "zeta_f32", "evd2_one_f32", "evd2_batched_f32",
    "upsilon", "gram", "rot", "step", "strategy_pairs", "strategy_is_checkpoint", "Fm",
    "gesvj", "gesvj_batched", "num_threads", "set_num_threads", "EVD_TAN", "EVD_NOBACKSCALE", "ZETA_ZERO",
    "norm_ef", "norm_ef_cols", "dgsscl",
    "OK", "ENOCONV", "EINVAL", "ENONFINITE", "ERANK",
]

OK, ENOCONV, EINVAL, ENONFINITE, ERANK = 0, 1, -1, -2, -3
EVD_TAN, EVD_NOBACKSCALE = 0x1, 0x2
ZETA_ZERO = 2**31 - 1

_D = ct.c_double
_PD = ct.POINTER(ct.c_double)
_I64 = ct.c_int64


class RSpec(ct.Structure):
    """Reduction spec R = (W, c, xor-offset sequence), R#15."""
    _fields_ = [("W", ct.c_int32), ("c", ct.c_int32), ("noffs", ct.c_int32),
                ("offs", ct.c_int32 * 32)]

    @classmethod
    def make(cls, W, c, offs):
        r = cls()
        r.W, r.c, r.noffs = int(W), int(c), len(offs)
        for k, o in enumerate(offs):
            r.offs[k] = int(o)
        return r

    def as_tuple(self):
        return (self.W, self.c, tuple(self.offs[k] for k in range(self.noffs)))


_lib = None


def lib():
    global _lib
    if _lib is None:
        path = build()
        L = ct.CDLL(path)
        L.orc_hypot.restype = _D
        L.orc_hypot.argtypes = [_D, _D]
        L.orc_zeta.restype = _D
        L.orc_zeta.argtypes = [_D, _D, _D, _D]
        _F, _PF = ct.c_float, ct.POINTER(ct.c_float)
        L.orc_hypot_f32.restype = _F
        L.orc_hypot_f32.argtypes = [_F, _F]
        L.orc_zeta_f32.restype = _F
        L.orc_zeta_f32.argtypes = [_F, _F, _F, _F]
        L.orc_evd2_one_f32.restype = None
        L.orc_evd2_one_f32.argtypes = [ct.c_int, _F, _F, _F, _F, ct.c_uint, _PF, _PF, _PF, _PF,
                                       _PF, ct.POINTER(ct.c_int32), ct.POINTER(ct.c_int)]
        L.orc_evd2_batched_f32.restype = ct.c_int
        L.orc_evd2_batched_f32.argtypes = [ct.c_int, _I64] + [ct.c_void_p] * 11 + [ct.c_uint]
        L.orc_evd2_one.restype = None
        L.orc_evd2_one.argtypes = [ct.c_int, _D, _D, _D, _D, ct.c_uint, _PD, _PD, _PD, _PD, _PD,
                                   ct.POINTER(ct.c_int32), ct.POINTER(ct.c_int)]
        L.orc_evd2_batched.restype = ct.c_int
        L.orc_evd2_batched.argtypes = [ct.c_int, _I64] + [ct.c_void_p] * 11 + [ct.c_uint]
        L.orc_colnorm.restype = None
        L.orc_colnorm.argtypes = [ct.c_int, _I64, ct.c_void_p, ct.POINTER(RSpec), _PD, _PD]
        L.orc_dot.restype = None
        L.orc_dot.argtypes = [ct.c_int, _I64, ct.c_void_p, _D, _D, ct.c_void_p, _D, _D,
                              ct.POINTER(RSpec), _PD, _PD]
        L.orc_cvg.restype = ct.c_int
        L.orc_cvg.argtypes = [_D, _D, _D]
        L.orc_upsilon.restype = _D
        L.orc_upsilon.argtypes = [_I64]
        L.orc_gram.restype = None
        L.orc_gram.argtypes = [_D] * 6 + [_PD] * 4
        L.orc_rot.restype = _D
        L.orc_rot.argtypes = [ct.c_int, _I64, ct.c_void_p, ct.c_void_p, _D, _D, _D]
        L.orc_step.restype = ct.c_int
        L.orc_step.argtypes = [ct.c_int, _I64, _I64, _I64, ct.c_void_p, _I64, ct.c_void_p, _I64,
                               ct.c_void_p, _I64, _D, ct.POINTER(RSpec), ct.c_void_p,
                               ct.c_void_p, ct.POINTER(_I64), _PD]
        L.orc_strategy_pairs.restype = ct.c_int
        L.orc_strategy_pairs.argtypes = [_I64, _I64, _I64, ct.c_void_p]
        L.orc_strategy_is_checkpoint.restype = ct.c_int
        L.orc_strategy_is_checkpoint.argtypes = [_I64, _I64, _I64]
        L.orc_Fm.restype = ct.c_int
        L.orc_Fm.argtypes = [ct.c_int, _I64]
        L.orc_gesvj.restype = ct.c_int
        L.orc_gesvj.argtypes = [ct.c_int, _I64, _I64, ct.c_void_p, _I64, ct.c_void_p, _I64,
                                ct.c_void_p, ct.c_void_p, ct.c_void_p, _I64, ct.c_int32,
                                ct.POINTER(ct.c_int32), ct.c_void_p, ct.c_int32,
                                ct.POINTER(ct.c_int32), ct.POINTER(RSpec)]
        L.orc_gesvj_batched.restype = ct.c_int
        L.orc_gesvj_batched.argtypes = [ct.c_int, _I64, _I64, _I64, ct.c_void_p, _I64, _I64,
                                        ct.c_void_p, _I64, _I64, ct.c_void_p, ct.c_int32,
                                        ct.c_void_p, ct.c_void_p, ct.c_int32, ct.c_void_p,
                                        ct.POINTER(RSpec)]
        L.orc_norm_ef.restype = ct.c_int
        L.orc_norm_ef.argtypes = [ct.c_int, _I64, ct.c_void_p, ct.c_int, ct.c_int, _PD, _PD, _PD,
                                  _PD]
        L.orc_dgsscl.restype = None
        L.orc_dgsscl.argtypes = [_I64, ct.c_void_p, ct.c_void_p, _D, _D, _D, _D, _D]
        L.orc_set_num_threads.restype = None
        L.orc_set_num_threads.argtypes = [ct.c_int]
        L.orc_num_threads.restype = ct.c_int
        L.orc_num_threads.argtypes = []
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ct.c_void_p)


def _f64(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a


def num_threads():
    return lib().orc_num_threads()


def set_num_threads(t):
    """OpenMP threads of the batched entry points (timing only)."""
    lib().orc_set_num_threads(int(t))


def hypot(x, y):
    return lib().orc_hypot(float(x), float(y))


def zeta(a11, a22, re, im=0.0):
    return lib().orc_zeta(float(a11), float(a22), float(re), float(im))


def evd2_one(is_complex, a11, a22, re, im=0.0, flags=0):
    out = [_D() for _ in range(5)]
    z, p = ct.c_int32(), ct.c_int()
    lib().orc_evd2_one(int(bool(is_complex)), float(a11), float(a22), float(re), float(im),
                       flags, *[ct.byref(o) for o in out], ct.byref(z), ct.byref(p))
    l1, l2, c, sr, si = (o.value for o in out)
    return dict(lam1=l1, lam2=l2, cos=c, sin_re=sr, sin_im=si, zeta=z.value, perm=p.value)


def hypot_f32(x, y):
    return float(np.float32(lib().orc_hypot_f32(np.float32(x), np.float32(y))))


def zeta_f32(a11, a22, re, im=0.0):
    return lib().orc_zeta_f32(*[np.float32(v) for v in (a11, a22, re, im)])


def evd2_one_f32(is_complex, a11, a22, re, im=0.0, flags=0):
    out = [ct.c_float() for _ in range(5)]
    z, p = ct.c_int32(), ct.c_int()
    lib().orc_evd2_one_f32(int(bool(is_complex)), *[float(np.float32(v)) for v in (a11, a22, re, im)],
                           flags, *[ct.byref(o) for o in out], ct.byref(z), ct.byref(p))
    l1, l2, c, sr, si = (np.float32(o.value) for o in out)
    return dict(lam1=l1, lam2=l2, cos=c, sin_re=sr, sin_im=si, zeta=z.value, perm=p.value)


def _f32(x):
    return np.ascontiguousarray(x, dtype=np.float32)


def evd2_batched_f32(a11, a22, a21_re, a21_im=None, flags=0):
    """Single-precision batched EVD.  Complex iff a21_im is given."""
    cplx = a21_im is not None
    a11, a22, re = _f32(a11), _f32(a22), _f32(a21_re)
    im = _f32(a21_im) if cplx else None
    r = a11.shape[0]
    out = {k: np.empty(r, np.float32) for k in ("lam1", "lam2", "cos", "sin_re")}
    out["sin_im"] = np.empty(r, np.float32) if cplx else None
    out["zeta"] = np.empty(r, np.int32)
    out["perm"] = np.empty((r + 31) // 32, np.uint32)
    p = lambda a: None if a is None else a.ctypes.data_as(ct.c_void_p)  # noqa: E731
    st = lib().orc_evd2_batched_f32(int(cplx), r, p(a11), p(a22), p(re), p(im), p(out["lam1"]),
                                    p(out["lam2"]), p(out["cos"]), p(out["sin_re"]),
                                    p(out["sin_im"]), p(out["zeta"]), p(out["perm"]), flags)
    if st != OK:
        raise ValueError(f"orc_evd2_batched_f32 status {st}")
    return out


def evd2_batched(a11, a22, a21_re, a21_im=None, flags=0):
    """Batched EVD (Alg 2.3 / SM2.2).  Complex iff a21_im is given."""
    cplx = a21_im is not None
    a11, a22, re = _f64(a11), _f64(a22), _f64(a21_re)
    im = _f64(a21_im) if cplx else None
    r = a11.shape[0]
    out = {k: np.empty(r, np.float64) for k in ("lam1", "lam2", "cos", "sin_re")}
    out["sin_im"] = np.empty(r, np.float64) if cplx else None
    out["zeta"] = np.empty(r, np.int32)
    out["perm"] = np.empty((r + 31) // 32, np.uint32)
    st = lib().orc_evd2_batched(int(cplx), r, _ptr(a11), _ptr(a22), _ptr(re), _ptr(im),
                                _ptr(out["lam1"]), _ptr(out["lam2"]), _ptr(out["cos"]),
                                _ptr(out["sin_re"]), _ptr(out["sin_im"]), _ptr(out["zeta"]),
                                _ptr(out["perm"]), flags)
    if st != OK:
        raise ValueError(f"orc_evd2_batched status {st}")
    return out


def _as_cols(x):
    """column vector -> (is_complex, float64 view with interleaved re/im)."""
    x = np.ascontiguousarray(x)
    if np.iscomplexobj(x):
        return 1, x.astype(np.complex128).view(np.float64), x.shape[0]
    return 0, x.astype(np.float64), x.shape[0]


def colnorm(x, R):
    c, xf, m = _as_cols(x)
    e, f = _D(), _D()
    lib().orc_colnorm(c, m, _ptr(xf), ct.byref(R), ct.byref(e), ct.byref(f))
    return e.value, f.value


def dot(xq, eq, fq, xp, ep, fp, R):
    c, q, m = _as_cols(xq)
    _, p, _ = _as_cols(xp)
    zr, zi = _D(), _D()
    lib().orc_dot(c, m, _ptr(q), eq, fq, _ptr(p), ep, fp, ct.byref(R), ct.byref(zr), ct.byref(zi))
    return zr.value, zi.value


def cvg(zre, zim, ups):
    return bool(lib().orc_cvg(zre, zim, ups))


def upsilon(m):
    return lib().orc_upsilon(int(m))


def gram(zre, zim, e1, f1, e2, f2):
    o = [_D() for _ in range(4)]
    lib().orc_gram(zre, zim, e1, f1, e2, f2, *[ct.byref(v) for v in o])
    return tuple(v.value for v in o)


def rot(xp, xq, c, C, S=0.0):
    """In-place rotation of two 1-D columns (numpy float64 or complex128)."""
    cplx = np.iscomplexobj(xp)
    assert xp.flags.c_contiguous and xq.flags.c_contiguous
    a = xp.view(np.float64) if cplx else xp
    b = xq.view(np.float64) if cplx else xq
    return lib().orc_rot(int(cplx), xp.shape[0], _ptr(a), _ptr(b), c, C, S)


def _mat_view(A):
    """Fortran-ordered (m, n) numpy -> (cplx, float64 buffer, ld)."""
    assert A.flags.f_contiguous, "matrices are column-major (Fortran order)"
    cplx = np.iscomplexobj(A)
    buf = A.reshape(-1, order="F").view(np.float64) if cplx else A.reshape(-1, order="F")
    return int(cplx), buf, A.shape[0]


def step(G, V, pairs, R, tol=0.0):
    """One step in place on Fortran-ordered G (m x ncols) and V (nv x ncols)."""
    cplx, gb, ldg = _mat_view(G)
    _, vb, ldv = _mat_view(V) if V is not None else (cplx, None, G.shape[1])
    m, n = G.shape
    nv = V.shape[0] if V is not None else n
    pairs = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1)
    ce = np.zeros(n, np.float64)
    cf = np.zeros(n, np.float64)
    t = _I64(0)
    M = _D(0.0)
    st = lib().orc_step(cplx, m, n, nv, _ptr(gb), ldg, _ptr(vb), ldv, _ptr(pairs), pairs.size // 2,
                        tol, ct.byref(R), _ptr(ce), _ptr(cf), ct.byref(t), ct.byref(M))
    if st != OK:
        raise ValueError(f"orc_step status {st}")
    return dict(col_e=ce, col_f=cf, t=t.value, mmax=M.value)


def strategy_pairs(n, B, step_idx):
    out = np.empty(n, np.int32)
    st = lib().orc_strategy_pairs(n, B, step_idx, _ptr(out))
    if st != OK:
        raise ValueError(f"orc_strategy_pairs status {st}")
    return out.reshape(-1, 2)


def strategy_is_checkpoint(n, B, step_idx):
    return bool(lib().orc_strategy_is_checkpoint(n, B, step_idx))


def Fm(cplx, m):
    return lib().orc_Fm(int(cplx), int(m))


def gesvj(A, R, B=None, max_sweeps=30, s0_adjust=0):
    """Full SVD (Alg 4.1).  A: (m, n) numpy, any order.  Returns dict(U, V,
    sigma, sigma_e, sigma_f, sweeps, tps, status, scale).  status 0: U
    normalised, sigma = Sigma sorted (R#24).  status 1 (ENOCONV, C = S): U
    holds the iteration matrix G = U Sigma' (scaled by 2^scale) and sigma /
    sigma_e / sigma_f hold Sigma' in column order (R#25).
    s0_adjust is added to s0 of Eq. (skn) (R#40)."""
    m, n = A.shape
    cplx = np.iscomplexobj(A)
    dt = np.complex128 if cplx else np.float64
    G = np.asfortranarray(A.astype(dt, copy=True))
    V = np.zeros((n, n), dt, order="F")
    c, gb, lda = _mat_view(G)
    _, vb, ldv = _mat_view(V)
    sig = np.zeros(n)
    se = np.zeros(n)
    sf = np.zeros(n)
    sw = ct.c_int32(0)
    sc = ct.c_int32(0)
    tps = np.zeros(max(max_sweeps, 1), np.int64)
    B = n if B is None else B
    st = lib().orc_gesvj(c, m, n, _ptr(gb), lda, _ptr(vb), ldv, _ptr(sig), _ptr(se), _ptr(sf), B,
                         max_sweeps, ct.byref(sw), _ptr(tps), int(s0_adjust), ct.byref(sc),
                         ct.byref(R))
    if st < 0:
        raise ValueError(f"orc_gesvj status {st}")
    return dict(U=G, V=V, sigma=sig, sigma_e=se, sigma_f=sf, sweeps=sw.value,
                tps=tps[:sw.value], status=st, scale=sc.value)


def gesvj_batched(A, R, max_sweeps=30, s0_adjust=0):
    """A: (batch, m, n) numpy; each matrix column-major in the returned U."""
    b, m, n = A.shape
    cplx = np.iscomplexobj(A)
    dt = np.complex128 if cplx else np.float64
    # column-major per matrix: store as (batch, n, m) C-order == each matrix F-order
    G = np.ascontiguousarray(np.transpose(A.astype(dt), (0, 2, 1)))
    V = np.zeros((b, n, n), dt)
    sig = np.zeros((b, n))
    sw = np.zeros(b, np.int32)
    st = np.zeros(b, np.int32)
    sc = np.zeros(b, np.int32)
    gb = G.view(np.float64) if cplx else G
    vb = V.view(np.float64) if cplx else V
    lib().orc_gesvj_batched(int(cplx), b, m, n, _ptr(gb), m, m * n, _ptr(vb), n, n * n,
                            _ptr(sig), max_sweeps, _ptr(sw), _ptr(st), int(s0_adjust), _ptr(sc),
                            ct.byref(R))
    U = np.transpose(G, (0, 2, 1))
    Vm = np.transpose(V, (0, 2, 1))
    return dict(U=U, V=Vm, sigma=sig, sweeps=sw, status=st, scale=sc)


def norm_ef(x, s=32, reduction=0):
    """NEXT-3: ||x||_F by the one-pass (e, f) method of Alg SM6.3
    with s lanes (R#35-R#38).  x: 1-D float64 or complex128.  reduction 0:
    pairwise (Eq. redj), 1: sequential (Eq. reds).  Returns (e'', f'', e, f):
    ||x|| = 2^e'' f'' and ||x||^2 = 2^e f."""
    x = np.ascontiguousarray(x)
    cplx = np.iscomplexobj(x)
    x = x.astype(np.complex128 if cplx else np.float64)
    e, f, e2, f2 = (ct.c_double() for _ in range(4))
    st = lib().orc_norm_ef(int(cplx), x.shape[0], _ptr(x), s, reduction, ct.byref(e), ct.byref(f),
                           ct.byref(e2), ct.byref(f2))
    if st != 0:
        raise ValueError("orc_norm_ef: invalid arguments")
    return e.value, f.value, e2.value, f2.value


def norm_ef_cols(A, s=32, reduction=0):
    """norm_ef of every column of the 2-D array A: arrays (e'', f'')."""
    n = A.shape[1]
    out = [norm_ef(A[:, j], s, reduction) for j in range(n)]
    return np.array([o[0] for o in out]), np.array([o[1] for o in out])


def dgsscl(gp, gq, ep, fp, eq, fq, a21):
    """NEXT-4: real Gram-Schmidt orthogonalization of g_q against g_p, Alg SM8.1 /
    Eq. (DGS) (R#39).  Returns the new g_q."""
    gp = np.ascontiguousarray(gp, dtype=np.float64)
    out = np.array(gq, dtype=np.float64, copy=True)
    lib().orc_dgsscl(gp.shape[0], _ptr(gp), _ptr(out), ep, fp, eq, fq, a21)
    return out
