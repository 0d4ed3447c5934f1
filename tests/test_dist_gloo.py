"""Multi-rank (N > 1) host logic on CPU: world-size-2 `gloo` process groups.

The GPU path runs one rank per GPU with NCCL; what can be checked
without GPUs is the decomposition it relies on:
  * r-slab split + slab-exact input generation (each rank builds only its planes),
  * one halo plane per side suffices for the 27-point anisotropic operator and the
    7-point isotropic one (rows of a slab touch only planes i0-1 .. i0+nl),
  * PCG with per-rank partial dot products summed by an all-reduce (the library's
    reduction protocol) reproduces the single-domain iterates and iteration count,
  * bench.py's max-over-ranks timing and uid broadcast helpers.
The oracle supplies the matrix; the halo exchange and reductions are gloo.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(fn, world=2, *args):
    port = _free_port()
    mp.spawn(_entry, args=(world, port, fn, args), nprocs=world, join=True)


def _entry(rank, world, port, fn, args):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------
def _slab_inputs(rank, world):
    import workloads as W
    shape = (14, 10, 16)
    i0, nl = W.split_planes(shape[0], world)[rank]
    full = W.make_config("c4_scale512", shape=shape)
    part = W.make_config("c4_scale512", shape=shape, slab=(i0, nl))
    for key in ("T", "rho"):
        assert torch.equal(part[key], full[key][i0:i0 + nl]), key
    assert torch.equal(part["b"], full["b"][:, i0:i0 + nl])
    assert torch.equal(part["v"], full["v"][:, i0:i0 + nl])
    for a, b in zip(part["visc_faces"], full["visc_faces"]):
        assert torch.equal(a, b[i0:i0 + nl])
    # the slabs tile the grid, rank order = r order
    got = [None] * world
    dist.all_gather_object(got, (i0, nl))
    assert got[0][0] == 0 and all(got[r][0] + got[r][1] == got[r + 1][0] for r in range(world - 1))
    assert sum(n for _, n in got) == shape[0]


@pytest.mark.parametrize("world", [2])
def test_slab_exact_inputs(world):
    _run(_slab_inputs, world)


# ----------------------------------------------------------------------------
def _exchange(x_local, nl, plane, rank, world):
    """[nl*plane] local vector -> [(nl+2)*plane] with lo/hi halo planes (zeros at walls)."""
    lo = torch.zeros(plane, dtype=torch.float64)
    hi = torch.zeros(plane, dtype=torch.float64)
    reqs = []
    if rank > 0:
        reqs.append(dist.isend(x_local[:plane].clone(), rank - 1))
        reqs.append(dist.irecv(lo, rank - 1))
    if rank < world - 1:
        reqs.append(dist.isend(x_local[-plane:].clone(), rank + 1))
        reqs.append(dist.irecv(hi, rank + 1))
    for r in reqs:
        r.wait()
    return torch.cat([lo, x_local, hi])


def _dist_pcg(rank, world, aniso):
    import workloads as W
    from oracle import core as O
    shape = (12, 9, 14)
    g = W.spherical_grid(*shape)
    cfg = W.make_config("c1_spitzer64", shape=shape)
    T = cfg["T"].numpy()
    kap = O.spitzer_face_kappa(g, T, cfg["kappa0"], cfg["T_cut"])
    op = O.Operator(g, kap, cfg["b"].numpy() if aniso else None)
    dt = 50.0 * O.dt_euler(op)
    A = O.be_system(op, dt).tocsr()
    rhs = op.WV * T.ravel()
    n1, n2, n3 = shape
    plane = n2 * n3
    i0, nl = W.split_planes(n1, world)[rank]
    rows = slice(i0 * plane, (i0 + nl) * plane)
    # halo depth: the slab's rows touch only planes i0-1 .. i0+nl
    Ar = A[rows]
    cols = Ar.nonzero()[1]
    assert cols.min() >= max(i0 - 1, 0) * plane and cols.max() < min(i0 + nl + 1, n1) * plane
    lo_c = (i0 - 1) * plane
    ext = np.arange(lo_c, (i0 + nl + 1) * plane)
    valid = (ext >= 0) & (ext < n1 * plane)
    A_ext = Ar[:, ext[valid]]

    def matvec(p_local):
        pe = _exchange(torch.as_tensor(p_local), nl, plane, rank, world).numpy()
        return A_ext @ pe[valid]

    def dot(a, b):
        t = torch.tensor([float(a @ b)], dtype=torch.float64)   # per-rank partial
        dist.all_reduce(t)                                        # summed across ranks
        return float(t.item())

    # PAPER.md Fig. 1 with point-Jacobi PC1, x0 = u^n, stop on r.z <= rtol^2 b.P^-1 b (DESIGN R8)
    b = rhs[rows]
    x = T.ravel()[rows].copy()
    P = A.diagonal()[rows]
    r = b - matvec(x)
    z = r / P
    p = z.copy()
    rz = dot(r, z)
    thresh = 1e-24 * dot(b, b / P)
    k = 0
    while rz > thresh and k < 10000:
        k += 1
        y = matvec(p)
        alpha = rz / dot(p, y)
        x += alpha * p
        r -= alpha * y
        z = r / P
        rz_old, rz = rz, dot(r, z)
        if rz <= thresh:
            break
        p = z + (rz / rz_old) * p
    ref, it = O.be_pcg_solve(op, T, dt, rtol=1e-12)
    assert abs(k - it[0]) <= 1, (k, it)
    xs = [None] * world
    dist.all_gather_object(xs, x)
    xg = np.concatenate(xs)
    # a residual-stopped iterate is unique only to ~cond(A) rtol: the distributed one must be
    # as close to the single-domain oracle as that is to the exact solve
    import scipy.sparse.linalg as spl
    exact = spl.spsolve(A.tocsc(), rhs)
    tol = max(1e-11, np.linalg.norm(ref.ravel() - exact) / np.linalg.norm(exact))
    assert np.linalg.norm(xg - ref.ravel()) <= tol * np.linalg.norm(ref)


@pytest.mark.parametrize("aniso", [True, False])
def test_distributed_pcg_matches_single_domain(aniso):
    _run(_dist_pcg, 2, aniso)


# ----------------------------------------------------------------------------
def _dist_pcg_merged(rank, world, aniso):
    """The library's default merged iteration on r-slabs: per iteration ONE halo
    exchange of z, w, p (their boundary planes) and ONE all-reduce of the four
    partial sums r.z, p.y, z.y, w.y per rank."""
    import workloads as W
    from oracle import core as O
    shape = (12, 9, 14)
    g = W.spherical_grid(*shape)
    cfg = W.make_config("c1_spitzer64", shape=shape)
    T = cfg["T"].numpy()
    kap = O.spitzer_face_kappa(g, T, cfg["kappa0"], cfg["T_cut"])
    op = O.Operator(g, kap, cfg["b"].numpy() if aniso else None)
    dt = 50.0 * O.dt_euler(op)
    A = O.be_system(op, dt).tocsr()
    rhs = op.WV * T.ravel()
    n1, n2, n3 = shape
    plane = n2 * n3
    i0, nl = W.split_planes(n1, world)[rank]
    rows = slice(i0 * plane, (i0 + nl) * plane)
    ext = np.arange((i0 - 1) * plane, (i0 + nl + 1) * plane)
    valid = (ext >= 0) & (ext < n1 * plane)
    A_ext = A[rows][:, ext[valid]]
    d = 1.0 / A.diagonal()[rows]
    n_allreduce = 0

    def halo(v):
        return _exchange(torch.as_tensor(v), nl, plane, rank, world).numpy()[valid]

    def allreduce(vals):
        nonlocal n_allreduce
        n_allreduce += 1
        t = torch.tensor(vals, dtype=torch.float64)
        dist.all_reduce(t)
        return t.tolist()

    b = rhs[rows]
    x = T.ravel()[rows].copy()
    z = (b - A_ext @ halo(x)) * d
    thresh = 1e-24 * allreduce([float(b @ (b * d))])[0]
    rz0 = allreduce([float(np.sum(z * z / d))])[0]
    k = 0
    if rz0 > thresh:
        w = p = None
        alpha = beta = 0.0
        while k < 10000:
            k += 1
            if k > 1:
                # the pass forms z_k and p_k at every staged position (own + halo planes):
                # exchanging z, w, p of the previous iteration is all it needs
                zh, wh, ph = halo(z), halo(w), halo(p)
                z = z - alpha * w
                x = x + alpha * p
                p = z + beta * p
                pe = zh - alpha * wh
                pe = pe + beta * ph
            else:
                p = z.copy()
                pe = halo(p)
            y = A_ext @ pe
            w = d * y
            rz, pAp, zy, wy = allreduce([float(np.sum(z * z / d)), float(p @ y), float(z @ y), float(w @ y)])
            alpha = rz / pAp
            rz_next = rz - 2.0 * alpha * zy + alpha * alpha * wy
            if rz_next <= thresh:
                x = x + alpha * p
                break
            beta = rz_next / rz
    ref, it = O.be_pcg_solve(op, T, dt, rtol=1e-12)
    assert abs(k - it[0]) <= 1, (k, it)
    assert n_allreduce == k + 2          # one per iteration (+ the two of the initial residual)
    xs = [None] * world
    dist.all_gather_object(xs, x)
    xg = np.concatenate(xs)
    import scipy.sparse.linalg as spl
    exact = spl.spsolve(A.tocsc(), rhs)
    tol = max(1e-11, np.linalg.norm(ref.ravel() - exact) / np.linalg.norm(exact))
    assert np.linalg.norm(xg - ref.ravel()) <= 2 * tol * np.linalg.norm(ref)   # DESIGN R12


@pytest.mark.parametrize("aniso", [True, False])
def test_distributed_merged_pcg_matches_single_domain(aniso):
    _run(_dist_pcg_merged, 2, aniso)


# ----------------------------------------------------------------------------
def _bench_helpers(rank, world):
    import bench
    dev = torch.device("cpu")
    v = bench.allreduce_max(float(rank + 1) * 10.0, dev, world)
    assert v == 10.0 * world
    obj = [b"uid-bytes-from-rank0" if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    assert obj[0] == b"uid-bytes-from-rank0"


def test_bench_max_over_ranks_and_uid_broadcast():
    _run(_bench_helpers, 2)
