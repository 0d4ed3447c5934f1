"""ctypes wrapper of the plain-C oracle (oracle/c/sts_oracle.c) -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__ (build / smoke) and bench.py's cpu_baseline may use it.
It shares no code with paper_1610_01265_b200/.  Functions take numpy arrays and a
workloads.Grid-like object (geom, x1f..x3c, periodic3).
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(_HERE, "c", "sts_oracle.c")
LIB = os.path.join(_HERE, "c", "libsts_oracle.so")
_lib = None


def build(force=False):
    """Compile the C oracle (gcc -O2, plain C11, OpenMP for the full-grid checker; no CUDA)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.run(["gcc", "-O2", "-std=c11", "-fopenmp", "-shared", "-fPIC", "-o", LIB + ".tmp", SRC, "-lm"],
                       check=True)
        os.replace(LIB + ".tmp", LIB)
    return LIB


class _Grid(ctypes.Structure):
    _fields_ = [("n1", ctypes.c_int), ("n2", ctypes.c_int), ("n3", ctypes.c_int), ("periodic3", ctypes.c_int),
                ("spherical", ctypes.c_int)] + [(n, ctypes.c_void_p) for n in ("x1f", "x1c", "x2f", "x2c", "x3f", "x3c")]


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        P, D, I = ctypes.c_void_p, ctypes.c_double, ctypes.c_int
        G = ctypes.POINTER(_Grid)
        L.oc_face_kappa.argtypes = [G, P, D, D, D, D, P, P, P]
        L.oc_op_apply.argtypes = [G, I, I, P, P, P, P, P, P, P]
        L.oc_dt_euler.argtypes = [G, I, P, P, P, P, P]
        L.oc_dt_euler.restype = D
        L.oc_rkl2_num_stages.argtypes = [D, D]
        L.oc_rkl2_num_stages.restype = I
        L.oc_rkl2_advance.argtypes = [G, I, I, P, P, P, P, P, P, D, I, P]
        L.oc_be_pcg.argtypes = [G, I, I, P, P, P, P, P, P, D, D, I, P, P]
        L.oc_be_pcg.restype = I
        L.oc_check_full.argtypes = [G, I, I, P, P, P, P, P, P, P, D, P, P]
        L.oc_set_threads.argtypes = [I]
        L.oc_max_threads.restype = I
        _lib = L
    return _lib


class CGrid:
    def __init__(self, g):
        self._keep = [np.ascontiguousarray(a, dtype=np.float64) for a in (g.x1f, g.x1c, g.x2f, g.x2c, g.x3f, g.x3c)]
        n1, n2, n3 = len(self._keep[1]), len(self._keep[3]), len(self._keep[5])
        self.shape = (n1, n2, n3)
        self.s = _Grid(n1, n2, n3, int(bool(g.periodic3)), int(g.geom == "spherical"),
                       *[a.ctypes.data for a in self._keep])

    @property
    def ptr(self):
        return ctypes.byref(self.s)


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _c(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def face_kappa(g, T, kappa0, T_cut, fc_r0=10.0, fc_w=0.0):
    G = CGrid(g)
    T = _c(T)
    k = [np.zeros(G.shape) for _ in range(3)]
    lib().oc_face_kappa(G.ptr, _p(T), kappa0, T_cut, fc_r0, fc_w, *[_p(x) for x in k])
    return k


def _args(kap, b, w):
    kap = [_c(x) for x in kap]
    return kap, _c(b), _c(w), (0 if b is None else 1)


def op_apply(g, u, kap, b=None, w=None):
    G = CGrid(g)
    kap, b, w, mode = _args(kap, b, w)
    u = _c(u)
    ncomp = 1 if u.ndim == 3 else u.shape[0]
    out = np.zeros_like(u)
    lib().oc_op_apply(G.ptr, mode, ncomp, *[_p(x) for x in kap], _p(b), _p(w), _p(u), _p(out))
    return out


def dt_euler(g, kap, b=None, w=None):
    G = CGrid(g)
    kap, b, w, mode = _args(kap, b, w)
    return lib().oc_dt_euler(G.ptr, mode, *[_p(x) for x in kap], _p(b), _p(w))


def rkl2_num_stages(dt, dt_exp):
    return lib().oc_rkl2_num_stages(float(dt), float(dt_exp))


def rkl2_advance(g, u0, kap, b, w, dt, s):
    G = CGrid(g)
    kap, b, w, mode = _args(kap, b, w)
    u0 = _c(u0)
    ncomp = 1 if u0.ndim == 3 else u0.shape[0]
    out = np.zeros_like(u0)
    lib().oc_rkl2_advance(G.ptr, mode, ncomp, *[_p(x) for x in kap], _p(b), _p(w), _p(u0), float(dt), int(s),
                          _p(out))
    return out


def be_pcg_solve(g, un, kap, b, w, dt, rtol=1e-12, kmax=100000):
    G = CGrid(g)
    kap, b, w, mode = _args(kap, b, w)
    un = _c(un)
    ncomp = 1 if un.ndim == 3 else un.shape[0]
    x = np.zeros_like(un)
    it = (ctypes.c_int * ncomp)()
    lib().oc_be_pcg(G.ptr, mode, ncomp, *[_p(a) for a in kap], _p(b), _p(w), _p(un), float(dt), float(rtol),
                    int(kmax), _p(x), it)
    return x, list(it)


def set_threads(n):
    """OpenMP threads of the oracle's parallel loops (face kappa, full-grid checker)."""
    lib().oc_set_threads(int(n))


def max_threads():
    return lib().oc_max_threads()


def check_full(g, un, kap, b, w, x, dt):
    """Matrix-free full-grid check of a backward-Euler iterate (oc_check_full): per
    component (sum r^2/A_ii, sum rhs^2/A_ii, max|r|/max|rhs|) for A = wV - dt L,
    rhs = wV un, r = rhs - A x, and the Gershgorin lambda_max of M = L/(wV).
    x None: only lambda_max.  Returns (list of per-component tuples, lambda_max)."""
    G = CGrid(g)
    kap, b, w, mode = _args(kap, b, w)
    un = _c(un)
    ncomp = 1 if un is None or un.ndim == 3 else un.shape[0]
    x = _c(x)
    out = np.zeros(4 * ncomp)
    lam = ctypes.c_double()
    lib().oc_check_full(G.ptr, mode, ncomp, *[_p(a) for a in kap], _p(b), _p(w), _p(un), _p(x), float(dt),
                        _p(out), ctypes.byref(lam))
    return [tuple(out[4 * c:4 * c + 3]) for c in range(ncomp)], lam.value
