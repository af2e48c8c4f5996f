"""CPU checks of the boundary: libjsvd.so loads and exports every symbol that
include/jsvd.h declares; the product package never imports the oracle."""
import ast
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "jsvd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(jsvd_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    syms = header_symbols()
    for s in ("jsvd_evd2_batched", "jsvd_sweep_step", "jsvd_gesvj"):
        assert s in syms


def test_library_builds_and_exports_every_header_symbol():
    from paper_2202_08361_b200 import _build
    lib = _build.build()
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (jsvd_\w+)", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing


def test_library_loads_and_answers_host_only_calls():
    import paper_2202_08361_b200 as J
    L = J.lib()
    assert J.status_string(0) == "JSVD_OK"
    assert "EINVAL" in J.status_string(-1)
    assert J.launch_count() >= 0
    # argument checks happen before any CUDA call
    assert L.jsvd_evd2_batched(0, -1, *([None] * 11), 0, None) == -1
    assert L.jsvd_evd2_batched(0, 0, *([None] * 11), 0, None) == 0


def test_host_pipeline_argument_checks_without_gpu():
    # jsvd_evd2_batched_host / jsvd_gesvj_batched_host validate before any CUDA call
    import ctypes as ct
    import numpy as np
    import paper_2202_08361_b200 as J
    L = J.lib()
    b = ct.c_size_t()
    assert L.jsvd_evd2_host_workspace(1, 48, ct.byref(b)) == -1      # chunk not a multiple of 32
    assert L.jsvd_evd2_host_workspace(1, 1 << 20, ct.byref(b)) == 0
    per_slot_c64 = 9 * 8 * (1 << 20) + 4 * (1 << 20) + 4 * ((1 << 20) // 32)
    assert b.value == 3 * per_slot_c64
    assert L.jsvd_evd2_host_workspace(0, 1 << 20, ct.byref(b)) == 0
    assert b.value == 3 * (7 * 8 * (1 << 20) + 4 * (1 << 20) + 4 * ((1 << 20) // 32))
    x = np.zeros(64)
    p = ct.c_void_p(x.ctypes.data)
    args = [p] * 4 + [p] * 5 + [None, None]
    # workspace smaller than the query -> ENOMEM, nothing launched
    assert L.jsvd_evd2_batched_host(1, 64, *args, 0, 32, p, 16, None) == -6
    # r == 0 is a no-op; complex without a21_im -> EINVAL
    assert L.jsvd_evd2_batched_host(1, 0, *args, 0, 32, None, 0, None) == 0
    assert L.jsvd_evd2_batched_host(1, 64, *([p] * 3 + [None] + [p] * 5 + [None, None]), 0, 32,
                                    p, 1 << 30, None) == -1
    assert L.jsvd_gesvj_batched_host_workspace(2, 64, 32, 8, ct.byref(b)) == -1  # R32: SVD is fp64
    assert L.jsvd_gesvj_batched_host_workspace(1, 64, 32, 8, ct.byref(b)) == 0 and b.value > 0
    assert L.jsvd_gesvj_batched_host(1, 4, 64, 32, p, p, p, p, 30, None, None, None, 2, p, 16,
                                     None) == -6


def test_sm100a_code_in_library():
    from paper_2202_08361_b200 import _build
    lib = _build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2202_08361_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            p = os.path.join(dp, f)
            if f.endswith(".py"):
                tree = ast.parse(open(p).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert not any(a.name.split(".")[0] == "oracle" for a in node.names), p
                    if isinstance(node, ast.ImportFrom):
                        assert (node.module or "").split(".")[0] != "oracle", p
            if f.endswith((".cu", ".cuh", ".h", ".cpp")):
                assert "oracle" not in re.sub(r"//.*", "", open(p).read()).lower() or \
                    "#include" not in open(p).read().split("oracle")[0][-200:], p


def test_gpu_calls_fail_loudly_without_cuda():
    import torch
    import paper_2202_08361_b200 as J
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    x = torch.zeros(4, dtype=torch.float64)
    with pytest.raises(ValueError):
        J.evd2_batched(x, x, x)


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("m", [1, 64, 256, 4096, 8192, 32768, 65536, 131072])
def test_step_rspec_is_a_valid_reduction_spec(cplx, m):
    import paper_2202_08361_b200 as J
    if cplx and m > 65536:
        with pytest.raises(J.JsvdError):
            J.step_rspec(cplx, m)
        return
    W, c, offs = J.step_rspec(cplx, m)
    assert c == 1 and W >= 256 and W & (W - 1) == 0
    assert sorted(offs) == [1 << k for k in range(W.bit_length() - 1)]
    assert offs[:5] == (16, 8, 4, 2, 1)
    per_lane = -(-m // W)  # register rows, plus as many shared-memory rows past W = 2048
    assert per_lane <= (16 if cplx else 32)
    assert W <= 2048 or per_lane > (8 if cplx else 16) or m <= W * (8 if cplx else 16)
