"""The C-ABI library builds, loads and exports every symbol include/*.h declares
(CPU-only: no kernel is launched here)."""
import ctypes
import glob
import math
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = []
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names += re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__ as e
    e.build()
    from paper_1610_01265_b200 import sts
    return sts.lib()


def test_header_declares_the_boundary():
    names = _declared()
    for n in ["sts_op_apply", "rkl2_num_stages", "rkl2_advance", "be_pcg_solve", "sts_dt_euler",
              "sts_face_kappa_spitzer", "sts_grid_create", "sts_grid_destroy", "sts_comm_init",
              "sts_nccl_unique_id", "sts_last_error", "sts_version"]:
        assert n in names, n


def test_library_exports_every_declared_symbol(lib):
    from paper_1610_01265_b200 import sts
    raw = ctypes.CDLL(sts.LIB_PATH)
    for n in _declared():
        assert hasattr(raw, n), f"{n} declared in include/ but not exported"


def test_library_is_built_for_sm100a(lib):
    from paper_1610_01265_b200 import sts
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", sts.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_stage_count_host_function_matches_brute_force(lib):
    # host-side arithmetic of the ABI (no GPU): Eq. (5), DESIGN R5
    from paper_1610_01265_b200 import sts
    for ratio in [1e-6, 0.1, 1.0, 9.99, 10.0, 10.01, 50.0, 100.0, 300.0, 500.0, 1000.0, 1e4]:
        s = sts.rkl2_num_stages(ratio, 1.0)
        smin = next(t for t in range(2, 10000) if (t * t + t - 2) / 4.0 >= ratio * (1 - 1e-15))
        assert s == smin
    assert sts.rkl2_num_stages(100.0, 1.0, force_odd=True) == 21
    assert lib.rkl2_num_stages(1.0, 0.0, 0) < 0           # dt_exp <= 0 -> STS_ERR_ARG
    assert lib.rkl2_num_stages(math.nan, 1.0, 0) < 0


def test_errors_are_reported_not_raised_in_c(lib):
    from paper_1610_01265_b200 import sts
    h = ctypes.c_void_p()
    x = (ctypes.c_double * 3)(0.0, 1.0, 2.0)
    c = (ctypes.c_double * 2)(0.5, 1.5)
    # bad sizes: n1 = 0
    rc = lib.sts_grid_create(ctypes.byref(h), 0, 0, 2, 2, x, c, x, c, x, c, 0, 0, 0, 1, 0)
    assert rc == -1 and b"n1" in lib.sts_last_error()
    # non-monotone faces
    xb = (ctypes.c_double * 3)(0.0, 2.0, 1.0)
    rc = lib.sts_grid_create(ctypes.byref(h), 0, 2, 2, 2, xb, c, x, c, x, c, 0, 0, 2, 1, 0)
    assert rc == -1
    assert lib.sts_grid_destroy(None) == 0
