"""Thin ctypes binding of libsts_b200.so (include/sts_b200.h).

Argument marshalling only: every step of the path runs in the library's CUDA
kernels.  Arrays are torch tensors (float64, C-contiguous) on the grid's CUDA
device — or on the host (pinned or pageable), in which case the library stages
them (the end-to-end path timed by bench.py).  There is no CPU fallback: if the
shared library is missing or no CUDA device is visible, calls raise.
"""
from __future__ import annotations

import ctypes
import math
import os

import torch  # noqa: F401  (loads CUDA runtime + NCCL before the library)

_HERE = os.path.dirname(os.path.abspath(__file__))
# (STS_LIB: an A-B variant built in-tree by build.py --out=...; the default is the product build)
LIB_PATH = os.environ.get("STS_LIB") or os.path.join(_HERE, "libsts_b200.so")

STS_OK = 0
STS_ERR_NOT_CONVERGED = -4
STS_ERR_BREAKDOWN = -7
GEOM = {"cartesian": 0, "spherical": 1}
MODE = {"iso": 0, "aniso": 1}
UID_BYTES = 128
# kernel classes of sts_grid_timing (include/sts_b200.h STS_K_*)
KERNEL_CLASSES = ["face_kappa", "aniso_F", "aniso_rkl2_first", "aniso_rkl2_stage", "aniso_pcg_r0",
                  "aniso_pcg_ap", "aniso_gersh", "iso_F", "iso_rkl2_first", "iso_rkl2_stage", "iso_pcg_r0",
                  "iso_pcg_ap", "iso_gersh", "pcg_update", "pcg_pupdate", "pcg_reduce", "halo",
                  "vertex_coef", "aniso_pcg_s", "pcg_xfinal", "iso_pcg_s", "aniso_pcg_m", "iso_pcg_m",
                  "aniso_rkl2_dstage", "iso_rkl2_dstage"]

_lib = None


class StsError(RuntimeError):
    def __init__(self, fn, code, msg):
        super().__init__(f"{fn} failed ({code}): {msg}")
        self.code = code


def lib():
    """Load the shared library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a)")
    L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    P = ctypes.c_void_p
    D = ctypes.c_double
    I = ctypes.c_int
    sig = {
        "sts_version": (I, []),
        "sts_last_error": (ctypes.c_char_p, []),
        "sts_grid_create": (I, [ctypes.POINTER(P), I, I, I, I, P, P, P, P, P, P, I, I, I, I, I]),
        "sts_grid_destroy": (I, [P]),
        "sts_grid_workspace_bytes": (I, [P, ctypes.POINTER(ctypes.c_size_t)]),
        "sts_grid_kernel_launches": (I, [P, ctypes.POINTER(ctypes.c_longlong)]),
        "sts_grid_comm_counts": (I, [P, ctypes.POINTER(ctypes.c_longlong), ctypes.POINTER(ctypes.c_longlong)]),
        "sts_grid_pcg_xmodes": (I, [P, I, ctypes.POINTER(I), ctypes.POINTER(I)]),
        "sts_grid_set_timing": (I, [P, I]),
        "sts_grid_set_tma": (I, [P, I]),
        "sts_grid_set_graphs": (I, [P, I]),
        "sts_grid_set_pcg_merged": (I, [P, I]),
        "sts_grid_set_rkl2_deviation": (I, [P, I]),
        "sts_grid_set_halo_overlap": (I, [P, I]),
        "sts_grid_timing_reset": (I, [P]),
        "sts_grid_timing": (I, [P, I, ctypes.POINTER(ctypes.c_longlong), ctypes.POINTER(D)]),
        "sts_nccl_unique_id": (I, [P, ctypes.c_size_t]),
        "sts_comm_init": (I, [P, I, I, P, ctypes.c_size_t]),
        "sts_face_kappa_spitzer": (I, [P, P, P, P, P, D, D, D, D, P]),
        "sts_op_apply": (I, [P, I, I, P, P, P, P, P, P, P, P]),
        "sts_dt_euler": (I, [P, I, P, P, P, P, P, ctypes.POINTER(D), P]),
        "rkl2_num_stages": (I, [D, D, I]),
        "rkl2_advance": (I, [P, I, I, P, P, P, P, P, P, P, D, I, P]),
        "rkl2_advance_hybrid": (I, [P, I, I, P, P, P, P, P, P, P, D, D, D, I, I, ctypes.POINTER(I), P]),
        "be_pcg_solve": (I, [P, I, I, P, P, P, P, P, P, P, D, D, I, ctypes.POINTER(I), P]),
        "be_pcg_solve_async": (I, [P, I, I, P, P, P, P, P, P, P, D, D, I, ctypes.POINTER(I), ctypes.POINTER(I), P]),
        "sts_grid_bind_coeffs": (I, [P, I, P, P, P, P, P, P]),
        "sts_grid_unbind_coeffs": (I, [P, I]),
        "sts_grid_join": (I, [P, P]),
        "sts_grid_synchronize": (I, [P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(fn, code, allow=()):
    if code != STS_OK and code not in allow:
        raise StsError(fn, code, lib().sts_last_error().decode())
    return code


def _ptr(t):
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        raise TypeError("expected a torch.Tensor")
    if t.dtype != torch.float64 or not t.is_contiguous():
        raise TypeError("arrays must be contiguous float64 tensors")
    return ctypes.c_void_p(t.data_ptr())


def _kptrs(k):
    """k = (k1, k2, k3) tensors, or None for the resident (bound) coefficients."""
    if k is None:
        return (None, None, None)
    return tuple(_ptr(x) for x in k)


class PcgResult:
    """Iterations / status of an asynchronous solve, written when the stream reaches its end."""

    def __init__(self, ncomp):
        self._iters = (ctypes.c_int * ncomp)(*([-1] * ncomp))
        self._status = ctypes.c_int(1)

    @property
    def iters(self):
        return list(self._iters)

    @property
    def status(self):
        return self._status.value


def _np_ptr(a):
    return ctypes.c_void_p(a.ctypes.data)


def _stream(stream):
    if stream is None:
        if torch.cuda.is_available():
            return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        return None
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def version():
    return lib().sts_version()


def rkl2_num_stages(dt, dt_exp, force_odd=False):
    """PAPER.md:142 Eq. (5) (DESIGN R5) — computed by the library."""
    s = lib().rkl2_num_stages(float(dt), float(dt_exp), int(bool(force_odd)))
    _check("rkl2_num_stages", STS_OK if s >= 2 else s)
    return s


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(UID_BYTES)
    _check("sts_nccl_unique_id", lib().sts_nccl_unique_id(buf, UID_BYTES))
    return buf.raw


class Grid:
    """Handle to a (slab of a) logically rectangular grid living on one GPU."""

    def __init__(self, geom, x1f, x1c, x2f, x2c, x3f, x3c, periodic3, i0=0, nl=None, n_virtual=1, device=0):
        import numpy as np
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (x1f, x1c, x2f, x2c, x3f, x3c)]
        self._keep = arrs
        n1, n2, n3 = len(arrs[1]), len(arrs[3]), len(arrs[5])
        nl = n1 - i0 if nl is None else nl
        h = ctypes.c_void_p()
        _check("sts_grid_create", lib().sts_grid_create(
            ctypes.byref(h), GEOM[geom], n1, n2, n3, *[_np_ptr(a) for a in arrs],
            int(bool(periodic3)), int(i0), int(nl), int(n_virtual), int(device)))
        self._h = h
        self.shape_global = (n1, n2, n3)
        self.i0, self.nl = i0, nl
        self.shape = (nl, n2, n3)
        self.device = torch.device("cuda", device)
        # False: calls with host (CPU) tensors return with their outputs written back; True:
        # they return once enqueued (pinned memory) -- then join() + synchronize first
        self.async_host = False

    @classmethod
    def from_grid(cls, g, i0=0, nl=None, n_virtual=1, device=0):
        """Duck-typed: any object with geom, x1f..x3c, periodic3 attributes."""
        return cls(g.geom, g.x1f, g.x1c, g.x2f, g.x2c, g.x3f, g.x3c, g.periodic3,
                   i0=i0, nl=nl, n_virtual=n_virtual, device=device)

    def close(self):
        if getattr(self, "_h", None):
            lib().sts_grid_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ info
    @property
    def kernel_launches(self):
        v = ctypes.c_longlong()
        _check("sts_grid_kernel_launches", lib().sts_grid_kernel_launches(self._h, ctypes.byref(v)))
        return v.value

    @property
    def comm_counts(self):
        """(local halo-exchange events, global reductions) so far (Sec. 2.4)."""
        a, b = ctypes.c_longlong(), ctypes.c_longlong()
        _check("sts_grid_comm_counts", lib().sts_grid_comm_counts(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def pcg_xmodes(self, ncomp=1):
        """(skipped, caught_up) x-update passes per component of the last synchronous solve."""
        a, b = (ctypes.c_int * ncomp)(), (ctypes.c_int * ncomp)()
        _check("sts_grid_pcg_xmodes", lib().sts_grid_pcg_xmodes(self._h, int(ncomp), a, b))
        return list(a), list(b)

    @property
    def workspace_bytes(self):
        v = ctypes.c_size_t()
        _check("sts_grid_workspace_bytes", lib().sts_grid_workspace_bytes(self._h, ctypes.byref(v)))
        return v.value

    def set_timing(self, enable=True):
        _check("sts_grid_set_timing", lib().sts_grid_set_timing(self._h, int(bool(enable))))

    def set_tma(self, enable=True):
        """Use the TMA pipelined anisotropic kernels where eligible (default) or force the cp.async ones."""
        _check("sts_grid_set_tma", lib().sts_grid_set_tma(self._h, int(bool(enable))))

    def set_graphs(self, enable=True):
        """Replay PCG iteration pairs as CUDA graphs (default) or launch every kernel directly."""
        _check("sts_grid_set_graphs", lib().sts_grid_set_graphs(self._h, int(bool(enable))))

    def set_pcg_merged(self, enable=True):
        """One fused pass + one reduction per PCG iteration (default) or the two-pass S / U iteration."""
        _check("sts_grid_set_pcg_merged", lib().sts_grid_set_pcg_merged(self._h, int(bool(enable))))

    def set_rkl2_deviation(self, enable=True):
        """RKL2 stages 2..s-1 on the deviation D_j = Y_j - Y0 (default) or on Y_j as Fig. 2 prints them."""
        _check("sts_grid_set_rkl2_deviation", lib().sts_grid_set_rkl2_deviation(self._h, int(bool(enable))))

    def set_halo_overlap(self, enable=True):
        """Decomposed grids: overlap the halo exchange with the interior planes (one-plane
        boundary launches) or wait for it and run one launch per slab (default)."""
        _check("sts_grid_set_halo_overlap", lib().sts_grid_set_halo_overlap(self._h, int(bool(enable))))

    def timing_reset(self):
        _check("sts_grid_timing_reset", lib().sts_grid_timing_reset(self._h))

    def timing(self):
        """{class name: (launches, device ms)} since the last timing_reset()."""
        out = {}
        for i, name in enumerate(KERNEL_CLASSES):
            n = ctypes.c_longlong()
            ms = ctypes.c_double()
            _check("sts_grid_timing", lib().sts_grid_timing(self._h, i, ctypes.byref(n), ctypes.byref(ms)))
            out[name] = (n.value, ms.value)
        return out

    def bind_coeffs(self, mode, k=None, b=None, w=None, stream=None):
        """Bind `mode`'s coefficients (resident across calls; None keeps the bound array).
        Ops called with k=None then use them (include/sts_b200.h "Resident coefficients")."""
        k = k if k is not None else (None, None, None)
        self._bound = getattr(self, "_bound", {})
        keep = self._bound.setdefault(mode, {})   # device tensors are referenced: keep them alive
        for name, t in (("k1", k[0]), ("k2", k[1]), ("k3", k[2]), ("b", b), ("w", w)):
            if t is not None:
                keep[name] = t
        _check("sts_grid_bind_coeffs", lib().sts_grid_bind_coeffs(
            self._h, MODE[mode], *_kptrs(k), _ptr(b), _ptr(w), _stream(stream)))

    def unbind_coeffs(self, mode):
        _check("sts_grid_unbind_coeffs", lib().sts_grid_unbind_coeffs(self._h, MODE[mode]))
        getattr(self, "_bound", {}).pop(mode, None)

    def join(self, stream=None):
        """Make `stream` wait for the handle's outstanding host-array copies."""
        _check("sts_grid_join", lib().sts_grid_join(self._h, _stream(stream)))

    def synchronize(self):
        _check("sts_grid_synchronize", lib().sts_grid_synchronize(self._h))

    def _host_done(self, stream, *arrays):
        """Host (CPU) tensors make the C call asynchronous (pinned) -- unless the Grid is in
        async_host mode, wait here so that the outputs can be read on return."""
        if self.async_host:
            return
        if any(isinstance(a, torch.Tensor) and a.device.type == "cpu" for a in arrays if a is not None):
            self.join(stream)
            if stream is None:
                torch.cuda.current_stream(self.device).synchronize()
            elif hasattr(stream, "synchronize"):
                stream.synchronize()
            else:
                torch.cuda.synchronize(self.device)

    def comm_init(self, nranks, rank, uid: bytes):
        buf = ctypes.create_string_buffer(uid, UID_BYTES)
        _check("sts_comm_init", lib().sts_comm_init(self._h, int(nranks), int(rank), buf, UID_BYTES))

    # ------------------------------------------------------------------ ops
    def _alloc(self, ncomp, like):
        shape = self.shape if ncomp == 1 else (ncomp,) + self.shape
        dev = like.device if like is not None else self.device
        if dev.type == "cpu":
            return torch.empty(shape, dtype=torch.float64, pin_memory=torch.cuda.is_available())
        return torch.empty(shape, dtype=torch.float64, device=dev)

    def face_kappa_spitzer(self, T, kappa0, T_cut, fc_r0=10.0, fc_w=0.0, out=None, stream=None, resident=False):
        """Face diffusivities into `out` (allocated if None) -- or, resident=True, into
        library-owned arrays bound as the "aniso" coefficients (returns None)."""
        if resident:
            out = (None, None, None)
        else:
            out = out or tuple(self._alloc(1, T) for _ in range(3))
        _check("sts_face_kappa_spitzer", lib().sts_face_kappa_spitzer(
            self._h, _ptr(T), *[_ptr(o) for o in out], float(kappa0), float(T_cut), float(fc_r0),
            float(fc_w), _stream(stream)))
        self._host_done(stream, T, *(out if not resident else ()))
        return None if resident else out

    def op_apply(self, mode, u, k, b=None, w=None, out=None, stream=None):
        ncomp = 1 if u.dim() == 3 else u.shape[0]
        out = self._alloc(ncomp, u) if out is None else out
        _check("sts_op_apply", lib().sts_op_apply(
            self._h, MODE[mode], ncomp, _ptr(u), _ptr(out), *_kptrs(k), _ptr(b), _ptr(w),
            _stream(stream)))
        self._host_done(stream, u, out, b, w, *(k or ()))
        return out

    def dt_euler(self, mode, k, b=None, w=None, stream=None):
        dt = ctypes.c_double()
        _check("sts_dt_euler", lib().sts_dt_euler(
            self._h, MODE[mode], *_kptrs(k), _ptr(b), _ptr(w), ctypes.byref(dt), _stream(stream)))
        return dt.value

    def rkl2_advance(self, mode, u0, k, b=None, w=None, dt=0.0, s=2, out=None, stream=None):
        ncomp = 1 if u0.dim() == 3 else u0.shape[0]
        out = self._alloc(ncomp, u0) if out is None else out
        _check("rkl2_advance", lib().rkl2_advance(
            self._h, MODE[mode], ncomp, _ptr(u0), _ptr(out), *_kptrs(k), _ptr(b), _ptr(w),
            float(dt), int(s), _stream(stream)))
        self._host_done(stream, u0, out, b, w, *(k or ()))
        return out

    def rkl2_advance_hybrid(self, mode, u0, k, b=None, w=None, dt=0.0, dt_exp=1.0, euler_frac=0.25,
                            n_euler=None, n_sub=1, out=None, stream=None):
        """PAPER.md:341 remedies: explicit-Euler prefix over euler_frac*dt (n_euler None: the
        library's default sub-step dt_exp/2, which annihilates the highest mode) + n_sub RKL2
        sub-cycles.  Returns (u1, (n_euler, s))."""
        if n_euler is None:
            n_euler = -1
        ncomp = 1 if u0.dim() == 3 else u0.shape[0]
        out = self._alloc(ncomp, u0) if out is None else out
        st = (ctypes.c_int * 2)()
        _check("rkl2_advance_hybrid", lib().rkl2_advance_hybrid(
            self._h, MODE[mode], ncomp, _ptr(u0), _ptr(out), *_kptrs(k), _ptr(b), _ptr(w),
            float(dt), float(dt_exp), float(euler_frac), int(n_euler), int(n_sub), st, _stream(stream)))
        self._host_done(stream, u0, out, b, w, *(k or ()))
        return out, (st[0], st[1])

    def be_pcg_solve(self, mode, un, k, b=None, w=None, dt=0.0, rtol=1e-12, kmax=100000, out=None,
                     stream=None, allow_not_converged=False):
        ncomp = 1 if un.dim() == 3 else un.shape[0]
        out = self._alloc(ncomp, un) if out is None else out
        iters = (ctypes.c_int * ncomp)()
        _check("be_pcg_solve", lib().be_pcg_solve(
            self._h, MODE[mode], ncomp, _ptr(un), _ptr(out), *_kptrs(k), _ptr(b), _ptr(w),
            float(dt), float(rtol), int(kmax), iters, _stream(stream)),
            allow=(STS_ERR_NOT_CONVERGED,) if allow_not_converged else ())
        self._host_done(stream, un, out, b, w, *(k or ()))
        return out, list(iters)

    def be_pcg_solve_async(self, mode, un, k, b=None, w=None, dt=0.0, rtol=1e-12, kmax=100000, out=None,
                           stream=None):
        """Enqueue a solve without waiting (include/sts_b200.h be_pcg_solve_async).  Returns
        (out, result): result.iters / result.status are valid once the stream has passed the
        solve (e.g. after join + synchronize)."""
        ncomp = 1 if un.dim() == 3 else un.shape[0]
        out = self._alloc(ncomp, un) if out is None else out
        res = PcgResult(ncomp)
        # the library writes res when the stream reaches the end of the solve: keep it alive
        # until then even if the caller drops it (the last 256 results are held)
        self._inflight = getattr(self, "_inflight", [])[-255:] + [res]
        _check("be_pcg_solve_async", lib().be_pcg_solve_async(
            self._h, MODE[mode], ncomp, _ptr(un), _ptr(out), *_kptrs(k), _ptr(b), _ptr(w),
            float(dt), float(rtol), int(kmax), res._iters, ctypes.byref(res._status), _stream(stream)))
        return out, res


def inf():
    return math.inf
