"""paper_2202_08361_b200 -- B200-native hot path of arXiv 2202.08361.

Thin Python binding over the C ABI of ``libjsvd.so`` (``include/jsvd.h``): the
functions here only marshal torch CUDA tensors into pointers, sizes and the
current CUDA stream; every step of the method runs in the library's sm_100a
kernels.  There is no CPU fallback: if the library is missing or no CUDA
device is present, the calls raise.

Entry points (same names as the C ABI, minus the ``jsvd_`` prefix):
  evd2_batched  -- Alg 2.2/2.3, SM2.1/SM2.2 batched 2x2 EVD
  sweep_step    -- one parallel Jacobi step, Alg 4.1 lines 7-38
  gesvj         -- the full one-sided Jacobi SVD, Alg 4.1
  gesvj_batched -- a batch of small independent SVDs (BASELINE configs[3])
"""
import ctypes as ct
import os

import torch

from ._build import LIB

__all__ = ["Dist", "Transport", "GesvjOpts", "DIST_SELF_P2P", "nccl_unique_id", "nccl_comm_init",
           "nccl_comm_destroy", "dist_columns", "dist_local_pairs", "lib", "evd2_batched", "sweep_step", "step_rspec", "batched_rspec", "strategy_pairs", "gesvj",
           "gesvj_workspace", "gesvj_batched", "launch_count", "evd2_batched_host",
           "evd2_host_workspace", "gesvj_batched_host", "gesvj_batched_host_workspace", "gesvj_host", "gesvj_host_workspace", "norm_ef", "dgsscl", "JsvdError", "R64", "C64",
           "EVD_TAN", "EVD_NOBACKSCALE", "ZETA_ZERO", "status_string"]

R64, C64, R32, C32 = 0, 1, 2, 3
EVD_TAN, EVD_NOBACKSCALE = 0x1, 0x2
ZETA_ZERO = 2 ** 31 - 1
OK, ENOCONV = 0, 1


class JsvdError(RuntimeError):
    def __init__(self, status, where):
        super().__init__(f"{where}: {status_string(status)} ({status})")
        self.status = status


_lib = None
_vp, _i64, _i32, _d = ct.c_void_p, ct.c_int64, ct.c_int32, ct.c_double

# jsvd_transport callbacks (include/jsvd.h): host-staged sendrecv / allreduce / allgather
SENDRECV_FN = ct.CFUNCTYPE(ct.c_int, _vp, _i32, ct.POINTER(_i32), ct.POINTER(_i32),
                           ct.POINTER(_vp), ct.POINTER(_i64))
ALLREDUCE_FN = ct.CFUNCTYPE(ct.c_int, _vp, _vp, _i32, _i32)
ALLGATHER_FN = ct.CFUNCTYPE(ct.c_int, _vp, _vp, _vp, _i64)


class Transport(ct.Structure):
    _fields_ = [("ctx", _vp), ("sendrecv", SENDRECV_FN), ("allreduce", ALLREDUCE_FN),
                ("allgather", ALLGATHER_FN)]


class Dist(ct.Structure):
    _fields_ = [("nccl_comm", _vp), ("rank", _i32), ("nranks", _i32),
                ("xport", ct.POINTER(Transport)), ("flags", ct.c_uint32)]


class GesvjOpts(ct.Structure):
    _fields_ = [("s0_adjust", _i32), ("max_steps", _i32)]


DIST_SELF_P2P = 0x1


def lib():
    """Load libjsvd.so (built by __graft_entry__.build()); raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise RuntimeError(f"{LIB} is missing: run __graft_entry__.build() "
                               "(there is no CPU fallback)")
        L = ct.CDLL(LIB)
        L.jsvd_evd2_batched.restype = ct.c_int
        L.jsvd_evd2_batched.argtypes = [ct.c_int, _i64] + [_vp] * 11 + [ct.c_uint32, _vp]
        L.jsvd_evd2_batched_f32.restype = ct.c_int
        L.jsvd_evd2_batched_f32.argtypes = L.jsvd_evd2_batched.argtypes
        L.jsvd_sweep_step.restype = ct.c_int
        L.jsvd_sweep_step.argtypes = [ct.c_int, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _d,
                                      _vp, _vp, _vp, _vp, _vp]
        L.jsvd_step_rspec.restype = ct.c_int
        L.jsvd_step_rspec.argtypes = [ct.c_int, _i64] + [ct.POINTER(_i32)] * 2 + [_vp,
                                                                                   ct.POINTER(_i32)]
        L.jsvd_batched_rspec.restype = ct.c_int
        L.jsvd_batched_rspec.argtypes = L.jsvd_step_rspec.argtypes
        L.jsvd_strategy_pairs.restype = ct.c_int
        L.jsvd_strategy_pairs.argtypes = [_i64, _i32, _i64, _vp, _vp]
        L.jsvd_gesvj_workspace.restype = ct.c_int
        L.jsvd_gesvj_workspace.argtypes = [ct.c_int, _i64, _i64, _i32, ct.POINTER(Dist),
                                           ct.POINTER(ct.c_size_t)]
        L.jsvd_gesvj.restype = ct.c_int
        L.jsvd_gesvj.argtypes = [ct.c_int, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp,
                                 _i32, _i32, ct.POINTER(_i32), _vp, ct.POINTER(_i32),
                                 ct.POINTER(GesvjOpts), _vp, ct.c_size_t, ct.POINTER(Dist), _vp]
        L.jsvd_gesvj_batched.restype = ct.c_int
        L.jsvd_gesvj_batched.argtypes = [ct.c_int, _i64, _i64, _i64, _vp, _i64, _i64, _vp, _i64,
                                         _i64, _vp, _i32, _vp, _vp, _vp, _vp,
                                         ct.POINTER(GesvjOpts), _vp]
        L.jsvd_batched_phase_profile.restype = ct.c_int
        L.jsvd_batched_phase_profile.argtypes = [ct.c_int, _i64, _i64, _i64, _vp, _i64, _i64, _vp,
                                                 _i64, _i64, _vp, _i32, _vp, _vp]
        L.jsvd_nccl_unique_id.restype = ct.c_int
        L.jsvd_nccl_unique_id.argtypes = [_vp]
        L.jsvd_nccl_comm_init.restype = ct.c_int
        L.jsvd_nccl_comm_init.argtypes = [ct.POINTER(_vp), _i32, _vp, _i32]
        L.jsvd_nccl_comm_destroy.restype = ct.c_int
        L.jsvd_nccl_comm_destroy.argtypes = [_vp]
        L.jsvd_dist_columns.restype = ct.c_int
        L.jsvd_dist_columns.argtypes = [_i64, _i32, _i32, _i32, _vp]
        L.jsvd_dist_local_pairs.restype = ct.c_int
        L.jsvd_dist_local_pairs.argtypes = [_i64, _i32, _i32, _i32, _i64, _vp]
        L.jsvd_evd2_host_workspace.restype = ct.c_int
        L.jsvd_evd2_host_workspace.argtypes = [ct.c_int, _i64, ct.POINTER(ct.c_size_t)]
        L.jsvd_evd2_batched_host.restype = ct.c_int
        L.jsvd_evd2_batched_host.argtypes = ([ct.c_int, _i64] + [_vp] * 11 +
                                             [ct.c_uint32, _i64, _vp, ct.c_size_t, _vp])
        L.jsvd_gesvj_batched_host_workspace.restype = ct.c_int
        L.jsvd_gesvj_batched_host_workspace.argtypes = [ct.c_int, _i64, _i64, _i64,
                                                        ct.POINTER(ct.c_size_t)]
        L.jsvd_gesvj_batched_host.restype = ct.c_int
        L.jsvd_gesvj_batched_host.argtypes = ([ct.c_int, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _i32,
                                               _vp, _vp, _vp, _i64, _vp, ct.c_size_t, _vp])
        L.jsvd_gesvj_host_workspace.restype = ct.c_int
        L.jsvd_gesvj_host_workspace.argtypes = [ct.c_int, _i64, _i64, _i32, ct.POINTER(ct.c_size_t)]
        L.jsvd_gesvj_host.restype = ct.c_int
        L.jsvd_gesvj_host.argtypes = [ct.c_int, _i64, _i64, _vp, _i64, _vp, _vp, _vp, _i32, _i32,
                                      ct.POINTER(_i32), _vp, ct.POINTER(_i32), _vp, ct.c_size_t, _vp]
        L.jsvd_norm_ef.restype = ct.c_int
        L.jsvd_norm_ef.argtypes = [ct.c_int, _i64, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _vp]
        L.jsvd_dgsscl.restype = ct.c_int
        L.jsvd_dgsscl.argtypes = [_i64, _i64, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp]
        L.jsvd_copy16.restype = ct.c_int
        L.jsvd_copy16.argtypes = [_i64, _vp, _vp, _vp]
        L.jsvd_fp64_peak.restype = ct.c_int
        L.jsvd_fp64_peak.argtypes = [_i32, _i64, _vp, ct.POINTER(_i64), _vp]
        L.jsvd_maxnorm.restype = ct.c_int
        L.jsvd_maxnorm.argtypes = [ct.c_int, _i64, _i64, _vp, _i64, _vp, _vp]
        L.jsvd_scale.restype = ct.c_int
        L.jsvd_scale.argtypes = [ct.c_int, _i64, _i64, _vp, _i64, _i32, _vp]
        L.jsvd_colnorms.restype = ct.c_int
        L.jsvd_colnorms.argtypes = [ct.c_int, _i64, _i64, _vp, _i64, _vp, _vp, _vp]
        L.jsvd_normalize.restype = ct.c_int
        L.jsvd_normalize.argtypes = [ct.c_int, _i64, _i64, _vp, _i64, _vp, _vp, _vp]
        L.jsvd_status_string.restype = ct.c_char_p
        L.jsvd_status_string.argtypes = [ct.c_int]
        L.jsvd_launch_count.restype = _i64
        L.jsvd_launch_count.argtypes = []
        _lib = L
    return _lib


def status_string(s):
    return lib().jsvd_status_string(int(s)).decode()


def launch_count():
    return int(lib().jsvd_launch_count())


def _check(st, where, allow=(OK,)):
    if st not in allow:
        raise JsvdError(st, where)
    return st


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ct.c_void_p(stream.cuda_stream)


def _p(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("jsvd expects CUDA tensors (no CPU fallback)")
    return ct.c_void_p(t.data_ptr())


def _f64(t, name):
    if t.dtype != torch.float64 or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous float64 CUDA tensor")
    return t


def evd2_batched(a11, a22, a21_re, a21_im=None, flags=0, out=None, stream=None):
    """Batched EVD of 2x2 Hermitian (a21_im given) / symmetric matrices.

    a11, a22, a21_re, a21_im: float64 (jsvd_evd2_batched) or float32
    (jsvd_evd2_batched_f32) CUDA tensors of length r (SoA).
    Returns dict(lam1, lam2, cos, sin_re[, sin_im], zeta, perm); pass ``out`` (a
    dict of preallocated tensors with those keys) to avoid allocation.
    """
    cplx = a21_im is not None
    r = a11.numel()
    dt = a11.dtype
    if dt not in (torch.float64, torch.float32):
        raise ValueError("a11 must be a float64 or float32 CUDA tensor")
    for n_, t in (("a11", a11), ("a22", a22), ("a21_re", a21_re)) + ((("a21_im", a21_im),) if cplx else ()):
        if t.dtype != dt or not t.is_contiguous():
            raise ValueError(f"{n_} must be a contiguous {dt} CUDA tensor like a11")
        if t.numel() != r:
            raise ValueError("all input streams must have the same length")
    if out is None:
        dev = a11.device
        out = {k: torch.empty(r, dtype=dt, device=dev) for k in ("lam1", "lam2", "cos", "sin_re")}
        out["sin_im"] = torch.empty(r, dtype=dt, device=dev) if cplx else None
        out["zeta"] = torch.empty(r, dtype=torch.int32, device=dev)
        out["perm"] = torch.empty((r + 31) // 32, dtype=torch.int32, device=dev)
    if dt == torch.float64:
        fn, code, name = lib().jsvd_evd2_batched, C64 if cplx else R64, "jsvd_evd2_batched"
    else:
        fn, code, name = lib().jsvd_evd2_batched_f32, C32 if cplx else R32, "jsvd_evd2_batched_f32"
    st = fn(code, r, _p(a11), _p(a22), _p(a21_re), _p(a21_im), _p(out["lam1"]),
            _p(out["lam2"]), _p(out["cos"]), _p(out["sin_re"]), _p(out.get("sin_im")),
            _p(out.get("zeta")), _p(out.get("perm")), flags, _stream(stream))
    _check(st, name)
    return out


def _scratch(nbytes, stream):
    """A device workspace allocated on the current stream for use on `stream`:
    record_stream keeps the caching allocator from handing the block to other
    work on the current stream while `stream` (and the library's internal
    streams, which `stream` joins) may still use it."""
    work = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    if stream is not None and stream != torch.cuda.current_stream():
        work.record_stream(stream)
    return work


def _host(t, name, dtype):
    if t is None:
        return None
    if t.is_cuda or t.dtype != dtype or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous {dtype} HOST tensor (pinned for overlap)")
    return ct.c_void_p(t.data_ptr())


def evd2_host_workspace(dtype, cplx, chunk):
    b = ct.c_size_t()
    code = (C64 if cplx else R64) if dtype == torch.float64 else (C32 if cplx else R32)
    _check(lib().jsvd_evd2_host_workspace(code, chunk, ct.byref(b)), "jsvd_evd2_host_workspace")
    return b.value


def evd2_batched_host(a11, a22, a21_re, a21_im=None, flags=0, out=None, chunk=1 << 21,
                      work=None, stream=None):
    """evd2_batched on HOST tensors (jsvd_evd2_batched_host): chunked H2D /
    kernel / D2H pipelined over three internal streams.  Inputs and ``out``
    (same keys as evd2_batched; allocated pinned when None) live in host memory;
    ``work`` is a uint8 CUDA tensor of at least evd2_host_workspace() bytes.
    Asynchronous on ``stream``: synchronise it before reading ``out``."""
    cplx = a21_im is not None
    r, dt = a11.numel(), a11.dtype
    if dt not in (torch.float64, torch.float32):
        raise ValueError("a11 must be float64 or float32")
    if out is None:
        out = {k: torch.empty(r, dtype=dt, pin_memory=True) for k in ("lam1", "lam2", "cos", "sin_re")}
        out["sin_im"] = torch.empty(r, dtype=dt, pin_memory=True) if cplx else None
        out["zeta"] = torch.empty(r, dtype=torch.int32, pin_memory=True)
        out["perm"] = torch.empty((r + 31) // 32, dtype=torch.int32, pin_memory=True)
    ptrs = []
    for n_, t in (("a11", a11), ("a22", a22), ("a21_re", a21_re), ("a21_im", a21_im),
                  ("lam1", out["lam1"]), ("lam2", out["lam2"]), ("cos", out["cos"]),
                  ("sin_re", out["sin_re"]), ("sin_im", out.get("sin_im"))):
        if t is not None and t.numel() != r:
            raise ValueError(f"{n_} must have length {r}")
        ptrs.append(_host(t, n_, dt))
    ptrs.append(_host(out.get("zeta"), "zeta", torch.int32))
    ptrs.append(_host(out.get("perm"), "perm", torch.int32))
    wb = evd2_host_workspace(dt, cplx, chunk)
    if work is None:
        work = _scratch(wb, stream)
    if not work.is_cuda or work.numel() < wb:
        raise ValueError(f"work must be a CUDA uint8 tensor of >= {wb} bytes")
    code = (C64 if cplx else R64) if dt == torch.float64 else (C32 if cplx else R32)
    st = lib().jsvd_evd2_batched_host(code, r, *ptrs, flags, chunk, _p(work), work.numel(),
                                      _stream(stream))
    _check(st, "jsvd_evd2_batched_host")
    return out


def gesvj_batched_host_workspace(cplx, m, n, chunk):
    b = ct.c_size_t()
    _check(lib().jsvd_gesvj_batched_host_workspace(C64 if cplx else R64, m, n, chunk, ct.byref(b)),
           "jsvd_gesvj_batched_host_workspace")
    return b.value


def gesvj_batched_host(A, max_sweeps=30, out=None, chunk=4096, work=None, stream=None,
                       transforms=True):
    """gesvj_batched on HOST tensors (jsvd_gesvj_batched_host).  A: (batch, m, n)
    host tensor whose matrices are packed column-major (A.stride() == (m*n, 1, m));
    A is not modified.  Returns dict(U, V, sigma, sweeps, status[, transforms]) of
    host tensors (pinned when allocated here).  Asynchronous on ``stream``."""
    b, m, n = A.shape
    if A.dtype not in (torch.float64, torch.complex128) or A.is_cuda or \
            A.stride() != (m * n, 1, m):
        raise ValueError("A must be a host float64/complex128 tensor of packed column-major matrices")
    cplx = A.dtype == torch.complex128
    if out is None:
        out = dict(U=torch.empty((b, n, m), dtype=A.dtype, pin_memory=True).transpose(1, 2),
                   V=torch.empty((b, n, n), dtype=A.dtype, pin_memory=True).transpose(1, 2),
                   sigma=torch.empty((b, n), dtype=torch.float64, pin_memory=True),
                   sweeps=torch.empty(b, dtype=torch.int32, pin_memory=True),
                   status=torch.empty(b, dtype=torch.int32, pin_memory=True),
                   transforms=torch.empty(b, dtype=torch.int64, pin_memory=True) if transforms else None)
    for k, shp in (("U", (m * n, 1, m)), ("V", (n * n, 1, n))):
        if out[k].is_cuda or out[k].dtype != A.dtype or out[k].stride() != shp or \
                out[k].shape != (b, shp[2], n):
            raise ValueError(f"out[{k!r}] must be a host tensor of packed column-major matrices")
    wb = gesvj_batched_host_workspace(cplx, m, n, chunk)
    if work is None:
        work = _scratch(wb, stream)
    if not work.is_cuda or work.numel() < wb:
        raise ValueError(f"work must be a CUDA uint8 tensor of >= {wb} bytes")
    st = lib().jsvd_gesvj_batched_host(
        C64 if cplx else R64, b, m, n, ct.c_void_p(A.data_ptr()), ct.c_void_p(out["U"].data_ptr()),
        ct.c_void_p(out["V"].data_ptr()), _host(out["sigma"], "sigma", torch.float64), max_sweeps,
        _host(out.get("sweeps"), "sweeps", torch.int32), _host(out.get("status"), "status", torch.int32),
        _host(out.get("transforms"), "transforms", torch.int64), chunk, _p(work), work.numel(),
        _stream(stream))
    _check(st, "jsvd_gesvj_batched_host")
    return out


def gesvj_host_workspace(cplx, m, n, nblocks=None):
    b = ct.c_size_t()
    _check(lib().jsvd_gesvj_host_workspace(C64 if cplx else R64, m, n,
                                           n if nblocks is None else nblocks, ct.byref(b)),
           "jsvd_gesvj_host_workspace")
    return b.value


def gesvj_host(A, nblocks=None, max_sweeps=30, out=None, work=None, stream=None):
    """jsvd_gesvj on a HOST matrix (jsvd_gesvj_host): A (m x n, column-major
    host tensor, float64 or complex128) is not modified; returns dict(U, V,
    sigma, sweeps, tps, status, scale) of host tensors (pinned when allocated
    here)."""
    if A.is_cuda or A.dtype not in (torch.float64, torch.complex128) or A.dim() != 2:
        raise ValueError("A must be a 2-D float64/complex128 HOST tensor")
    m, n = A.shape
    if (m > 1 and A.stride(0) != 1) or (n > 1 and A.stride(1) < m):
        raise ValueError("A must be column-major (use A.T.contiguous().T)")
    lda = A.stride(1) if n > 1 else m
    cplx = A.dtype == torch.complex128
    if out is None:
        out = dict(U=torch.empty((n, m), dtype=A.dtype, pin_memory=True).T,
                   V=torch.empty((n, n), dtype=A.dtype, pin_memory=True).T,
                   sigma=torch.empty(n, dtype=torch.float64, pin_memory=True))
    nb = n if nblocks is None else nblocks
    wb = gesvj_host_workspace(cplx, m, n, nb)
    if work is None:
        work = _scratch(wb, stream)
    if not work.is_cuda or work.numel() < wb:
        raise ValueError(f"work must be a CUDA uint8 tensor of >= {wb} bytes")
    sw, sc = _i32(0), _i32(0)
    tps = (_i64 * max(max_sweeps, 1))()
    st = lib().jsvd_gesvj_host(C64 if cplx else R64, m, n, ct.c_void_p(A.data_ptr()), lda,
                               ct.c_void_p(out["U"].data_ptr()), ct.c_void_p(out["V"].data_ptr()),
                               ct.c_void_p(out["sigma"].data_ptr()), nb, max_sweeps, ct.byref(sw),
                               ct.cast(tps, _vp), ct.byref(sc), _p(work), work.numel(),
                               _stream(stream))
    _check(st, "jsvd_gesvj_host", allow=(OK, ENOCONV))
    out.update(sweeps=sw.value, tps=[tps[k] for k in range(sw.value)], status=st, scale=sc.value)
    return out


def step_rspec(cplx, m):
    """(W, c, offsets) of the step kernel the library picks for (dtype, m)."""
    W, c, no = _i32(), _i32(), _i32()
    offs = (_i32 * 32)()
    _check(lib().jsvd_step_rspec(C64 if cplx else R64, m, ct.byref(W), ct.byref(c),
                                 ct.cast(offs, _vp), ct.byref(no)), "jsvd_step_rspec")
    return W.value, c.value, tuple(offs[k] for k in range(no.value))


def batched_rspec(cplx, m):
    """(W, c, offsets) of jsvd_gesvj_batched's kernel."""
    W, c, no = _i32(), _i32(), _i32()
    offs = (_i32 * 32)()
    _check(lib().jsvd_batched_rspec(C64 if cplx else R64, m, ct.byref(W), ct.byref(c),
                                    ct.cast(offs, _vp), ct.byref(no)), "jsvd_batched_rspec")
    return W.value, c.value, tuple(offs[k] for k in range(no.value))


def strategy_pairs(n, nblocks, step, out=None, stream=None, device="cuda"):
    if out is None:
        out = torch.empty(n, dtype=torch.int32, device=device)
    _check(lib().jsvd_strategy_pairs(n, nblocks, step, _p(out), _stream(stream)),
           "jsvd_strategy_pairs")
    return out.view(-1, 2)


def _mat(t, name):
    """column-major (m, n) CUDA tensor (float64 or complex128) -> (cplx, ld)."""
    if t.dtype not in (torch.float64, torch.complex128):
        raise ValueError(f"{name} must be float64 or complex128")
    m, n = t.shape
    ld = t.stride(1) if n > 1 else m
    if (m > 1 and t.stride(0) != 1) or ld < m:
        raise ValueError(f"{name} must be column-major (use A.T.contiguous().T)")
    return t.dtype == torch.complex128, ld


def sweep_step(G, V, pairs, tol=0.0, col_e=None, col_f=None, t_dev=None, mmax_dev=None,
               stream=None):
    """One Jacobi step in place on column-major G (m x ncols) and V (n x ncols):
    V has as many columns as G (the columns a driver holds) and n rows (the
    order of the full V; n = ncols for an unsharded SVD)."""
    cplx, ldg = _mat(G, "G")
    m, n = G.shape
    ldv = n
    if V is not None:
        cv, ldv = _mat(V, "V")
        if cv != cplx or V.shape[1] != n or V.shape[0] < n:
            raise ValueError("V must be (n >= ncols) x ncols of G's dtype")
        n = V.shape[0]
    dev = G.device
    col_e = torch.empty(n, dtype=torch.float64, device=dev) if col_e is None else col_e
    col_f = torch.empty(n, dtype=torch.float64, device=dev) if col_f is None else col_f
    t_dev = torch.zeros(1, dtype=torch.int64, device=dev) if t_dev is None else t_dev
    mmax_dev = torch.zeros(1, dtype=torch.float64, device=dev) if mmax_dev is None else mmax_dev
    pairs = pairs.reshape(-1)
    if pairs.dtype != torch.int32 or not pairs.is_contiguous():
        raise ValueError("pairs must be contiguous int32")
    st = lib().jsvd_sweep_step(C64 if cplx else R64, m, n, _p(G), ldg, _p(V), ldv, _p(pairs),
                               pairs.numel() // 2, float(tol), _p(col_e), _p(col_f), _p(t_dev),
                               _p(mmax_dev), _stream(stream))
    _check(st, "jsvd_sweep_step")
    return dict(col_e=col_e, col_f=col_f, t=t_dev, mmax=mmax_dev)


def maxnorm(G, out=None, stream=None):
    """max |component| of column-major G into the device scalar `out` (max-reduced)."""
    cplx, ld = _mat(G, "G")
    m, n = G.shape
    out = torch.zeros(1, dtype=torch.float64, device=G.device) if out is None else out
    _check(lib().jsvd_maxnorm(C64 if cplx else R64, m, n, _p(G), ld, _p(out), _stream(stream)),
           "jsvd_maxnorm")
    return out


def scale(G, s, stream=None):
    """G <- 2^s G in place (one rounding per component)."""
    cplx, ld = _mat(G, "G")
    m, n = G.shape
    _check(lib().jsvd_scale(C64 if cplx else R64, m, n, _p(G), ld, int(s), _stream(stream)),
           "jsvd_scale")
    return G


def colnorms(G, col_e=None, col_f=None, stream=None):
    """(e, f) of every column of G, in the step kernel's reduction order."""
    cplx, ld = _mat(G, "G")
    m, n = G.shape
    col_e = torch.empty(n, dtype=torch.float64, device=G.device) if col_e is None else col_e
    col_f = torch.empty(n, dtype=torch.float64, device=G.device) if col_f is None else col_f
    _check(lib().jsvd_colnorms(C64 if cplx else R64, m, n, _p(G), ld, _p(col_e), _p(col_f),
                               _stream(stream)), "jsvd_colnorms")
    return col_e, col_f


def norm_ef(G, col_e=None, col_f=None, col_e2=None, col_f2=None, stream=None):
    """NEXT-3: ||g_j|| of every column of column-major G by the one-pass (e, f)
    method of Alg SM6.3 (s = 32 lanes, jsvd_norm_ef).  Returns (col_e, col_f)
    with ||g_j|| = 2^col_e col_f; pass col_e2/col_f2 tensors to also get the
    (e, f) of ||g_j||^2."""
    cplx, ld = _mat(G, "G")
    m, n = G.shape
    col_e = torch.empty(n, dtype=torch.float64, device=G.device) if col_e is None else col_e
    col_f = torch.empty(n, dtype=torch.float64, device=G.device) if col_f is None else col_f
    _check(lib().jsvd_norm_ef(C64 if cplx else R64, m, n, _p(G), ld, _p(col_e), _p(col_f),
                              _p(col_e2), _p(col_f2), _stream(stream)), "jsvd_norm_ef")
    return col_e, col_f


def dgsscl(G, pairs, col_e, col_f, a21, stream=None):
    """NEXT-4: real Gram-Schmidt orthogonalization (Alg SM8.1 / Eq. DGS,
    jsvd_dgsscl) of g_q against g_p for each pair, in place on column-major
    float64 G.  pairs: int32 (npairs, 2); col_e/col_f: the columns' norms
    (e, f); a21: float64 (npairs,) the pairs' scaled dots a21'."""
    cplx, ld = _mat(G, "G")
    if cplx:
        raise ValueError("dgsscl is real only (the paper's complex variant is not given)")
    m, n = G.shape
    pairs = pairs.reshape(-1)
    if pairs.dtype != torch.int32 or not pairs.is_contiguous():
        raise ValueError("pairs must be contiguous int32")
    _check(lib().jsvd_dgsscl(m, n, _p(G), ld, _p(pairs), pairs.numel() // 2, _p(col_e), _p(col_f),
                             _p(_f64(a21, "a21")), _stream(stream)), "jsvd_dgsscl")
    return G


def normalize(G, col_e, col_f, stream=None):
    """u_j = 2^-e_j g_j / f_j in place."""
    cplx, ld = _mat(G, "G")
    m, n = G.shape
    _check(lib().jsvd_normalize(C64 if cplx else R64, m, n, _p(G), ld, _p(col_e), _p(col_f),
                                _stream(stream)), "jsvd_normalize")
    return G


def _opts(s0_adjust, max_steps=0):
    return ct.byref(GesvjOpts(int(s0_adjust), int(max_steps))) if (s0_adjust or max_steps) else None


def gesvj_workspace(cplx, m, n, nblocks=None, dist=None):
    b = ct.c_size_t()
    _check(lib().jsvd_gesvj_workspace(C64 if cplx else R64, m, n, n if nblocks is None else nblocks,
                                      ct.byref(dist) if dist is not None else None, ct.byref(b)),
           "jsvd_gesvj_workspace")
    return b.value


def gesvj(A, nblocks=None, max_sweeps=30, V=None, work=None, stream=None, s0_adjust=0,
          dist=None, n=None, max_steps=0, out=None):
    """Alg 4.1 in place: A (column-major m x ncols) becomes U (converged) or
    G = U Sigma' (status ENOCONV).  Returns dict(U, V, sigma,
    sigma_e, sigma_f, perm, sweeps, tps, status, scale).

    dist (a Dist struct, see dist.py): this rank's columns of a sharded SVD of
    order n (A: m x n/nranks packed, V: n x n/nranks); sigma / perm are the
    global sorted values, U and V stay distributed.  max_steps > 0 stops after
    that many steps (timing a bounded run: ENOCONV, no finalize)."""
    cplx, lda = _mat(A, "A")
    m, ncols = A.shape
    n = ncols if dist is None else int(n)
    dev = A.device
    if V is None:
        V = torch.empty((ncols, n), dtype=A.dtype, device=dev).T
    _, ldv = _mat(V, "V")
    if V.shape != (n, ncols):
        raise ValueError(f"V must be {n} x {ncols}")
    if out is None:
        out = dict(sigma=torch.empty(n, dtype=torch.float64, device=dev),
                   sigma_e=torch.empty(n, dtype=torch.float64, device=dev),
                   sigma_f=torch.empty(n, dtype=torch.float64, device=dev),
                   perm=torch.empty(n, dtype=torch.int32, device=dev))
    sig, se, sf, perm = out["sigma"], out["sigma_e"], out["sigma_f"], out["perm"]
    nb = n if nblocks is None else nblocks
    wb = gesvj_workspace(cplx, m, n, nb, dist)
    if work is None or work.numel() < wb:
        work = torch.empty(max(wb, 1), dtype=torch.uint8, device=dev)
    sw, sc = _i32(0), _i32(0)
    tps = (_i64 * max(max_sweeps, 1))()
    st = lib().jsvd_gesvj(C64 if cplx else R64, m, n, _p(A), lda, _p(V), ldv, _p(sig), _p(se),
                          _p(sf), _p(perm), nb, max_sweeps, ct.byref(sw), ct.cast(tps, _vp),
                          ct.byref(sc), _opts(s0_adjust, max_steps), _p(work), work.numel(),
                          ct.byref(dist) if dist is not None else None, _stream(stream))
    _check(st, "jsvd_gesvj", allow=(OK, ENOCONV))
    return dict(U=A, V=V, sigma=sig, sigma_e=se, sigma_f=sf, perm=perm, sweeps=sw.value,
                tps=[tps[k] for k in range(sw.value)], status=st, scale=sc.value)


def gesvj_batched(A, max_sweeps=30, V=None, sigma=None, sweeps=None, status=None, stream=None,
                  transforms=None, scale=None, s0_adjust=0):
    """A: (batch, m, n) CUDA tensor whose matrices are column-major, i.e.
    A.stride() == (m*n, 1, m) (use X.transpose(1,2).contiguous().transpose(1,2)).
    In place: A becomes U (per matrix as gesvj: G = U Sigma' on ENOCONV).
    Returns dict(U, V, sigma, sweeps, status, transforms, scale) (transforms:
    int64 transformed pair-steps, scale: int32 final s -- only when a tensor
    is passed)."""
    b, m, n = A.shape
    if A.dtype not in (torch.float64, torch.complex128) or A.stride(1) != 1 or A.stride(2) < m:
        raise ValueError("A must be float64/complex128 with column-major matrices")
    cplx = A.dtype == torch.complex128
    dev = A.device
    if V is None:
        V = torch.empty((b, n, n), dtype=A.dtype, device=dev).transpose(1, 2)
    sigma = torch.empty((b, n), dtype=torch.float64, device=dev) if sigma is None else sigma
    sweeps = torch.empty(b, dtype=torch.int32, device=dev) if sweeps is None else sweeps
    status = torch.empty(b, dtype=torch.int32, device=dev) if status is None else status
    st = lib().jsvd_gesvj_batched(C64 if cplx else R64, b, m, n, _p(A), A.stride(2), A.stride(0),
                                  _p(V), V.stride(2), V.stride(0), _p(sigma), max_sweeps,
                                  _p(sweeps), _p(status),
                                  _p(transforms) if transforms is not None else None,
                                  _p(scale) if scale is not None else None, _opts(s0_adjust),
                                  _stream(stream))
    _check(st, "jsvd_gesvj_batched")
    return dict(U=A, V=V, sigma=sigma, sweeps=sweeps, status=status, transforms=transforms,
                scale=scale)


PHASES = ("A: norms + dot", "wait after A", "B: test, Gram, EVD (warp 0) / V rotation (others)",
          "wait after B", "C: G rotation", "wait after C", "rescale check, loads, line 41",
          "sweep loop")


def batched_phase_profile(A, max_sweeps=30, stream=None):
    """jsvd_batched_phase_profile on (batch, 64, n) column-major matrices (in
    place, as gesvj_batched): per-phase cycles of warp 0 and of the other
    warps, summed over the CTAs -- dict(warp0={phase: cycles}, others=...)."""
    b, m, n = A.shape
    cplx = A.dtype == torch.complex128
    V = torch.empty((b, n, n), dtype=A.dtype, device=A.device).transpose(1, 2)
    sig = torch.empty((b, n), dtype=torch.float64, device=A.device)
    prof = torch.zeros(16, dtype=torch.int64, device=A.device)
    _check(lib().jsvd_batched_phase_profile(C64 if cplx else R64, b, m, n, _p(A), A.stride(2),
                                            A.stride(0), _p(V), V.stride(2), V.stride(0), _p(sig),
                                            max_sweeps, _p(prof), _stream(stream)),
           "jsvd_batched_phase_profile")
    p = prof.cpu().tolist()
    return dict(warp0=dict(zip(PHASES, p[:8])), others=dict(zip(PHASES, p[8:])))


def nccl_unique_id():
    """128-byte NCCL unique id (rank 0 creates it, every rank receives it)."""
    buf = (ct.c_char * 128)()
    _check(lib().jsvd_nccl_unique_id(ct.cast(buf, _vp)), "jsvd_nccl_unique_id")
    return bytes(buf)


def nccl_comm_init(nranks, uid, rank):
    """An NCCL communicator on the current device, owned by the caller
    (jsvd_nccl_comm_destroy)."""
    c = _vp()
    buf = (ct.c_char * 128).from_buffer_copy(uid)
    _check(lib().jsvd_nccl_comm_init(ct.byref(c), nranks, ct.cast(buf, _vp), rank),
           "jsvd_nccl_comm_init")
    return c.value


def nccl_comm_destroy(comm):
    _check(lib().jsvd_nccl_comm_destroy(comm), "jsvd_nccl_comm_destroy")


def dist_columns(n, nblocks, rank, nranks):
    """Global columns of rank `rank`'s local columns (jsvd_dist_columns); host."""
    out = (_i32 * (n // nranks))()
    _check(lib().jsvd_dist_columns(n, nblocks, rank, nranks, ct.cast(out, _vp)), "jsvd_dist_columns")
    return list(out)


def dist_local_pairs(n, nblocks, rank, nranks, step):
    """Local (p, q) column pairs of rank `rank` in step `step` (jsvd_dist_local_pairs); host."""
    out = (_i32 * (n // nranks))()
    _check(lib().jsvd_dist_local_pairs(n, nblocks, rank, nranks, step, ct.cast(out, _vp)),
           "jsvd_dist_local_pairs")
    return [(out[2 * k], out[2 * k + 1]) for k in range(n // nranks // 2)]


def copy16(src, dst, stream=None):
    """jsvd_copy16: dst <- src (contiguous CUDA tensors of the same byte size,
    a multiple of 16 bytes), the EVD kernel's streaming access pattern."""
    if not (src.is_cuda and dst.is_cuda and src.is_contiguous() and dst.is_contiguous()):
        raise ValueError("copy16: contiguous CUDA tensors")
    nb = src.numel() * src.element_size()
    if nb != dst.numel() * dst.element_size() or nb % 16:
        raise ValueError("copy16: equal sizes, a multiple of 16 bytes")
    s = torch.cuda.current_stream() if stream is None else stream
    _check(lib().jsvd_copy16(nb // 16, _p(src), _p(dst), s.cuda_stream), "jsvd_copy16")


def fp64_peak(iters=4096, blocks=None, stream=None):
    """Measured FP64 pipe throughput (DFMA instructions per second, thread
    level) of jsvd_fp64_peak, timed with CUDA events on `stream`."""
    dev = torch.cuda.current_device()
    if blocks is None:
        blocks = 8 * torch.cuda.get_device_properties(dev).multi_processor_count
    out = torch.empty(blocks * 256, dtype=torch.float64, device="cuda")
    cnt = _i64()
    s = torch.cuda.current_stream() if stream is None else stream
    _check(lib().jsvd_fp64_peak(blocks, 64, _p(out), ct.byref(cnt), s.cuda_stream), "jsvd_fp64_peak")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    _check(lib().jsvd_fp64_peak(blocks, iters, _p(out), ct.byref(cnt), s.cuda_stream), "jsvd_fp64_peak")
    e1.record(s)
    s.synchronize()
    return cnt.value / (e0.elapsed_time(e1) / 1e3)
