"""Pins of the plain-C oracle (oracle/c/sts_oracle.c; BASELINE north_star asks for a
plain CPU C implementation) against the numpy oracle -- itself pinned by closed forms,
DCT-exact solutions, direct solves and paper values (tests/test_oracle_*.py) -- and
against closed forms directly.  CPU only."""
import math

import numpy as np
import pytest

import workloads as W
from oracle import c_oracle as C
from oracle import core as O

GRIDS = [("sph", (6, 7, 8), True), ("sph", (5, 6, 9), False), ("sph", (4, 3, 2), True), ("sph", (3, 4, 1), True),
         ("cart", (6, 5, 7), False), ("cart", (5, 4, 6), True)]


def _grid(kind, shape, periodic):
    if kind == "cart":
        g = W.uniform_cartesian(*shape)
        if periodic:
            g = W.Grid("cartesian", g.x1f, g.x2f, g.x3f, True, x1c=g.x1c, x2c=g.x2c, x3c=g.x3c)
        return g
    g = W.spherical_grid(*shape, r1=3.0, dr0=0.2)
    if not periodic:
        g = W.Grid("spherical", g.x1f, np.linspace(0.3, 2.8, shape[1] + 1), np.linspace(0.0, 1.5, shape[2] + 1), False)
    return g


def _inputs(g, seed, aniso):
    rng = np.random.default_rng(seed)
    T = 1.5e6 * (1 + 0.3 * rng.uniform(-1, 1, g.shape))
    kap = O.spitzer_face_kappa(g, T, 1e-9, 5e5)
    b = W.random_unit_b(g, seed=seed).numpy() if aniso else None
    w = None if aniso else rng.uniform(0.5, 2.0, g.shape)
    return T, kap, b, w


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("case", GRIDS)
@pytest.mark.parametrize("aniso", [False, True])
def test_c_oracle_matches_numpy_oracle(case, aniso):
    g = _grid(*case)
    T, kap, b, w = _inputs(g, 7, aniso)
    kc = C.face_kappa(g, T, 1e-9, 5e5)
    for a, e in zip(kc, kap):
        np.testing.assert_allclose(a, e, rtol=1e-13, atol=0)
    op = O.Operator(g, kap, b, w)
    assert rel(C.op_apply(g, T, kap, b, w), op.apply(T)) <= 1e-12
    dte = O.dt_euler(op)
    assert abs(C.dt_euler(g, kap, b, w) - dte) <= 1e-12 * dte
    dt = 40.0 * dte
    s = O.rkl2_num_stages(dt, dte)
    assert C.rkl2_num_stages(dt, dte) == s
    ref = O.rkl2_advance(lambda x: (op.M @ x.ravel()).reshape(x.shape), T, dt, s)
    assert rel(C.rkl2_advance(g, T, kap, b, w, dt, s), ref) <= 1e-12
    xr, itr = O.be_pcg_solve(op, T, dt, rtol=1e-12)
    xc, itc = C.be_pcg_solve(g, T, kap, b, w, dt, 1e-12)
    assert abs(itc[0] - itr[0]) <= 1
    assert rel(xc, xr) <= 1e-9


def test_c_oracle_vector_components_and_heat_closed_form():
    """3 components are independent solves; on the uniform Cartesian heat problem the
    Gershgorin bound is the closed form 12 kappa / h^2 (interior rows)."""
    g = W.uniform_cartesian(6, 6, 6)
    kap = [np.ones(g.shape)] * 3
    assert abs(C.dt_euler(g, kap) - 2.0 / 12.0) <= 1e-15
    rng = np.random.default_rng(1)
    v = rng.normal(size=(3,) + g.shape)
    w = rng.uniform(0.5, 2.0, g.shape)
    F = C.op_apply(g, v, kap, None, w)
    for c in range(3):
        np.testing.assert_allclose(F[c], C.op_apply(g, v[c], kap, None, w), rtol=0, atol=0)
    x, it = C.be_pcg_solve(g, v, kap, None, w, 3.0)
    for c in range(3):
        xc, ic = C.be_pcg_solve(g, v[c], kap, None, w, 3.0)
        np.testing.assert_array_equal(x[c], xc)
        assert it[c] == ic[0]


def test_c_stage_count_brute_force():
    for r in np.logspace(-1, 4, 200):
        smin = next(t for t in range(2, 100000) if (t * t + t - 2) / 4.0 >= r * (1 - 1e-15))
        assert C.rkl2_num_stages(r, 1.0) == smin
    assert (C.rkl2_num_stages(1, 1), C.rkl2_num_stages(100, 1), C.rkl2_num_stages(500, 1)) == (2, 20, 45)


@pytest.mark.parametrize("case", GRIDS)
def test_c_oracle_fc_branch_matches_numpy(case):
    """The f_c(r) factor of the C oracle's face diffusivity, with the
    half-value radius placed inside the grid, against the numpy oracle (itself pinned by
    hand values in test_oracle_operator.py::test_fc_*)."""
    g = _grid(*case)
    T, _, _, _ = _inputs(g, 3, False)
    r0 = float(np.median(g.x1c))
    kc = C.face_kappa(g, T, 1e-9, 5e5, r0, 0.3)
    ko = O.spitzer_face_kappa(g, T, 1e-9, 5e5, r0, 0.3)
    off = O.spitzer_face_kappa(g, T, 1e-9, 5e5)
    for a, e, o in zip(kc, ko, off):
        np.testing.assert_allclose(a, e, rtol=1e-13, atol=0)
    if g.geom == "spherical":
        assert any(np.any(e != o) for e, o in zip(ko, off))   # the profile is active


@pytest.mark.parametrize("case", GRIDS)
@pytest.mark.parametrize("aniso", [False, True])
def test_full_grid_checker_matches_assembled_system(case, aniso):
    """oc_check_full (row c of L gathered matrix-free from the vertices / faces around c)
    against the numpy oracle's assembled sparse system: the Gershgorin bound of App. B
     and the preconditioned residual norms of the BE system (DESIGN R7, R8)
    for a perturbed iterate, for the direct solution (residual at rounding level) and
    for 3 components."""
    g = _grid(*case)
    T, kap, b, w = _inputs(g, 11, aniso)
    op = O.Operator(g, kap, b, w)
    dte = O.dt_euler(op)
    dt = 30.0 * dte
    A = O.be_system(op, dt)
    D = A.diagonal()
    rng = np.random.default_rng(5)
    x = T * (1.0 + 1e-3 * rng.normal(size=g.shape))
    res, lam = C.check_full(g, T, kap, b, w, x, dt)
    assert abs(2.0 / lam - dte) <= 1e-13 * dte
    rhs = op.WV * T.ravel()
    r = rhs - A @ x.ravel()
    num, den, mx = res[0]
    assert abs(num - float(r @ (r / D))) <= 1e-10 * float(r @ (r / D))
    assert abs(den - float(rhs @ (rhs / D))) <= 1e-13 * den
    assert abs(mx - np.abs(r).max() / np.abs(rhs).max()) <= 1e-10 * mx
    import scipy.sparse.linalg as spl
    xe = spl.spsolve(A.tocsc(), rhs).reshape(g.shape)
    (num_e, den_e, _), = C.check_full(g, T, kap, b, w, xe, dt)[0]
    assert num_e <= 1e-26 * den_e
    v = np.stack([T, x, xe])
    res3, lam3 = C.check_full(g, v, kap, b, w, np.stack([xe, xe, x]), dt)
    assert lam3 == lam and res3[0][0] <= 1e-26 * res3[0][1]
    for q, xq in ((1, xe), (2, x)):
        rq = op.WV * v[q].ravel() - A @ xq.ravel()
        assert abs(res3[q][0] - float(rq @ (rq / D))) <= 1e-9 * float(rq @ (rq / D)) + 1e-26 * res3[q][1]
