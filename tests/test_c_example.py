"""The C ABI from plain C (examples/evd_c.c): it builds against include/jsvd.h
and libjsvd.so with gcc alone (CPU), and on a GPU it runs the device and the
host-buffer EVD entry points, which must agree bit for bit and reconstruct A."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2202_08361_b200")


def _build(out):
    cmd = ["gcc", "-O2", "-std=c11", os.path.join(ROOT, "examples", "evd_c.c"),
           "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include", "-L" + LIBDIR,
           "-ljsvd", "-L/usr/local/cuda/lib64", "-lcudart", "-lm", "-Wl,-rpath," + LIBDIR, "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_c_example_builds(tmp_path):
    _build(str(tmp_path / "evd_c"))


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    exe = str(tmp_path / "evd_c")
    _build(exe)
    r = subprocess.run([exe, "100003"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "bit-identical" in r.stdout
