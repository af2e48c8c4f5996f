"""The seeded input generators: shard invariance and the config recipes."""
import math

import numpy as np

import synth


def test_shard_slices_are_bit_identical():
    full = synth.evd_cfg2(10000)
    part = synth.evd_cfg2(2500, off=5000)
    for a, b in zip(full, part):
        assert np.array_equal(a[5000:7500].view(np.uint64), b.view(np.uint64))
    g = synth.svd_cfg4(6, seed=4)
    h = synth.svd_cfg4(2, seed=4, off=3)
    assert np.array_equal(g[3:5], h)


def test_cfg1_recipe():
    a11, a22, a21 = synth.evd_cfg1(1 << 18)
    allv = np.concatenate([a11, a22, a21])
    nz = allv[allv != 0]
    e = np.frexp(np.abs(nz))[1] - 1
    normal = (e >= -20) & (e <= 20)
    assert normal.mean() > 0.985
    assert set(np.unique(e[~normal])) <= set(range(-1074, -1021)) | {1020}
    zeros = (allv == 0).sum()
    assert 0.002 < zeros / (1 << 18) < 0.005  # ~1% special, 1/3 zeros
    sub = (np.abs(a21) < 2.2250738585072014e-308) & (a21 != 0)
    assert 0.002 < sub.mean() < 0.005


def test_cfg2_recipe():
    a11, a22, re, im = synth.evd_cfg2(1 << 18)
    sub = (np.abs(re) < 2.2250738585072014e-308) & (np.abs(im) < 2.2250738585072014e-308)
    assert 0.017 < sub.mean() < 0.023
    big = np.zeros(1 << 18, bool)
    for x in (a11, a22, re, im):
        big |= np.abs(x) >= 2.0 ** 1023
    assert 0.008 < big.mean() < 0.012
    e = np.frexp(np.abs(a11))[1] - 1
    assert e.min() >= -1000 and e.max() <= 1023


def test_gauss_moments():
    g = synth.gauss(1 << 20, seed=1)
    assert abs(g.mean()) < 0.01 and abs(g.std() - 1) < 0.01
    assert np.isfinite(g).all()


def test_cfg3_prescribed_sigma():
    A, sig = synth.svd_cfg3(m=128, n=32, seed=3)
    s = np.linalg.svd(A, compute_uv=False)
    assert np.allclose(s, sig, rtol=0, atol=1e-14)
    assert sig[0] == 1.0 and math.isclose(sig[-1], 1e-12)
