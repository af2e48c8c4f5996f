"""Seeded synthetic inputs shared by tests, oracle legs and bench.

Holds none of the method's arithmetic.  Counter-based (SplitMix64 over
(seed, stream, global index)), so shards are bit-identical to slices of the
full batch.  The recipes are stated in DESIGN.md ("Synthetic inputs") and
follow BASELINE.json's configs; the paper's own datasets
are not reproduced.
"""
import ctypes as ct
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csynth.c")
LIB = os.path.join(HERE, "libsynth.so")

SEEDS = {1: 42, 2: 7, 3: 3, 4: 4, 5: 5}


def build(force=False):
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.run(["gcc", "-O2", "-std=gnu11", "-fopenmp", "-fPIC", "-shared", SRC,
                        "-o", LIB + ".tmp", "-lm"], check=True)
        os.replace(LIB + ".tmp", LIB)
    return LIB


_lib = None


def _L():
    global _lib
    if _lib is None:
        L = ct.CDLL(build())
        u64, i64, vp = ct.c_uint64, ct.c_int64, ct.c_void_p
        L.synth_sm64.restype = u64
        L.synth_sm64.argtypes = [u64, u64, u64]
        L.synth_evd_cfg1.argtypes = [u64, i64, i64, vp, vp, vp]
        L.synth_evd_cfg2.argtypes = [u64, i64, i64, vp, vp, vp, vp]
        L.synth_evd_cfg1_f32.argtypes = [u64, i64, i64, vp, vp, vp]
        L.synth_evd_cfg2_f32.argtypes = [u64, i64, i64, vp, vp, vp, vp]
        L.synth_gauss.argtypes = [u64, u64, i64, i64, vp]
        L.synth_uniform.argtypes = [u64, u64, i64, i64, vp]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ct.c_void_p)


def sm64(seed, stream, idx):
    return _L().synth_sm64(seed, stream, idx)


def evd_cfg1(r, seed=SEEDS[1], off=0):
    """(a11, a22, a21) float64 arrays of length r: BASELINE configs[0]."""
    a = [np.empty(r, np.float64) for _ in range(3)]
    _L().synth_evd_cfg1(seed, off, r, *map(_p, a))
    return tuple(a)


def evd_cfg2(r, seed=SEEDS[2], off=0):
    """(a11, a22, re, im) float64 arrays of length r: BASELINE configs[1]."""
    a = [np.empty(r, np.float64) for _ in range(4)]
    _L().synth_evd_cfg2(seed, off, r, *map(_p, a))
    return tuple(a)


def evd_cfg1_f32(r, seed=SEEDS[1], off=0):
    """(a11, a22, a21) float32: the single-precision analogue of configs[0]."""
    a = [np.empty(r, np.float32) for _ in range(3)]
    _L().synth_evd_cfg1_f32(seed, off, r, *map(_p, a))
    return tuple(a)


def evd_cfg2_f32(r, seed=SEEDS[2], off=0):
    """(a11, a22, re, im) float32: the single-precision analogue of configs[1]."""
    a = [np.empty(r, np.float32) for _ in range(4)]
    _L().synth_evd_cfg2_f32(seed, off, r, *map(_p, a))
    return tuple(a)


def gauss(count, seed, stream=0, off=0):
    out = np.empty(count, np.float64)
    _L().synth_gauss(seed, stream, off, count, _p(out))
    return out


def uniform(count, seed, stream=0, off=0):
    out = np.empty(count, np.float64)
    _L().synth_uniform(seed, stream, off, count, _p(out))
    return out


def gauss_matrix(m, n, seed, stream=0, complex_=False):
    """(m, n) Fortran-ordered N(0,1) matrix (complex: independent re, im)."""
    if complex_:
        re = gauss(m * n, seed, stream)
        im = gauss(m * n, seed, stream + 1)
        return np.asfortranarray((re + 1j * im).reshape(n, m).T)
    return np.asfortranarray(gauss(m * n, seed, stream).reshape(n, m).T)


def haar_q(m, n, seed, stream, complex_=False):
    """Q factor of a Householder QR of an (m, n) Gaussian matrix (numpy/LAPACK)."""
    q, _ = np.linalg.qr(gauss_matrix(m, n, seed, stream, complex_))
    return q


def svd_cfg3(m=4096, n=1024, seed=SEEDS[3], kappa=1e12):
    """A = Q1 diag(sigma) Q2^T, sigma_i = kappa^{-(i-1)/(n-1)} (configs[2])."""
    sig = kappa ** (-np.arange(n) / (n - 1))
    q1 = haar_q(m, n, seed, 0)
    q2 = haar_q(n, n, seed, 2)
    return np.asfortranarray((q1 * sig) @ q2.T), sig


def svd_cfg5(m=32768, n=8192, seed=SEEDS[5], log_range=8.0):
    """A = Q1 diag(sigma) Q2^H complex, sigma_i = 10^{-8 u_i} (configs[4])."""
    sig = 10.0 ** (-log_range * uniform(n, seed, 9))
    q1 = haar_q(m, n, seed, 0, True)
    q2 = haar_q(n, n, seed, 2, True)
    return np.asfortranarray((q1 * sig) @ q2.conj().T), sig


def svd_cfg5_torch(m=32768, n=8192, seed=SEEDS[5], log_range=8.0, device="cuda"):
    """configs[4] generated on the GPU with torch (QR + GEMM would take hours in
    numpy): A = Q1 diag(sigma) Q2^H, Q from torch.linalg.qr of complex Gaussian
    matrices drawn by this module's counter-based generator; sigma = 10^{-8 u}.
    Returns (A as an (m, n) column-major complex128 CUDA tensor, sigma numpy)."""
    import torch
    sig = 10.0 ** (-log_range * uniform(n, seed, 9))

    def cgauss(r, c, stream):
        re = torch.from_numpy(gauss(r * c, seed, stream)).to(device)
        im = torch.from_numpy(gauss(r * c, seed, stream + 1)).to(device)
        return torch.complex(re, im).reshape(c, r).T  # column-major (r, c) view

    q1, _ = torch.linalg.qr(cgauss(m, n, 0))
    q2, _ = torch.linalg.qr(cgauss(n, n, 2))
    A = (q1 * torch.from_numpy(sig).to(device)) @ q2.conj().T
    At = A.T.contiguous()  # (n, m) row-major == (m, n) column-major
    del q1, q2, A
    return At.T, sig


def svd_cfg4(batch, m=64, n=32, seed=SEEDS[4], off=0):
    """(batch, m, n) complex128; entries re, im ~ N(0,1) i.i.d. (configs[3]).
    Matrix b's column-major (re, im) stream starts at global element b*m*n."""
    cnt = batch * m * n
    re = gauss(cnt, seed, 0, off * m * n)
    im = gauss(cnt, seed, 1, off * m * n)
    z = (re + 1j * im).reshape(batch, n, m)
    return np.transpose(z, (0, 2, 1))
