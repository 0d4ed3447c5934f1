"""The boundary is a plain C ABI: examples/c_abi_demo.c (C, no Python, no PyTorch)
compiles against include/sts_b200.h and libsts_b200.so with gcc, and on a GPU runs a
heat-equation RKL2 advance and a BE + Jacobi-PCG solve on cudaMalloc'd arrays,
checking conservation of the total (PAPER.md:329 test problem, zero-flux walls)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1610_01265_b200")
CUDA = "/usr/local/cuda"


def _build(tmp_path):
    from paper_1610_01265_b200 import build as B
    B.build(verbose=False)
    exe = str(tmp_path / "c_abi_demo")
    cmd = ["gcc", "-O2", "-Wall", "-Werror", "-std=c11", os.path.join(ROOT, "examples", "c_abi_demo.c"),
           f"-I{ROOT}/include", f"-I{CUDA}/include", f"-L{LIBDIR}", "-lsts_b200", f"-L{CUDA}/lib64", "-lcudart",
           "-lm", f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_demo_compiles_as_c(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_c_demo_runs(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "c_abi_demo ok" in r.stdout
