"""Pins for the oracle's Gershgorin bound, RKL2 advance and BE+PCG solve.

Config 0 (BASELINE.json configs[0]): the isotropic constant-diffusivity heat
equation on a uniform Cartesian 32^3 grid with zero-flux walls is diagonalised
exactly by the DCT-II (scipy.fft), so RKL2 (closed-form Legendre amplification)
and BE (1/(1-z)) have exact discrete solutions; the analytic heat kernel with
image sources checks the continuum limit; tiny grids are solved densely.
"""
import math

import numpy as np
import pytest
import scipy.fft as sfft
from numpy.polynomial import legendre

import workloads as W
from oracle import core as O


def _R(s, z):
    bs = (s * s + s - 2.0) / (2.0 * s * (s + 1.0))
    w1 = 4.0 / (s * s + s - 2.0)
    return 1.0 - bs + bs * legendre.legval(1.0 + w1 * z, [0] * s + [1])


def _dct_lambda(n, h=1.0):
    lam1 = -(4.0 / h ** 2) * np.sin(np.pi * np.arange(n) / (2 * n)) ** 2
    return lam1[:, None, None] + lam1[None, :, None] + lam1[None, None, :]


@pytest.fixture(scope="module")
def heat():
    cfg = W.make_config("c0_heat32")
    g = cfg["grid"]
    op = O.Operator(g, [f.numpy() for f in cfg["faces"]])
    return cfg, g, op


def test_gershgorin_closed_form_cartesian(heat):
    _, g, op = heat
    # interior row of the 7-point Laplacian, kappa = h = 1: |diag| + 6 = 12
    assert abs(O.dt_euler(op) - 2.0 / 12.0) < 1e-15


def test_rkl2_config0_matches_dct_exact(heat):
    cfg, g, op = heat
    u0 = cfg["u"].numpy()
    dt_exp = O.dt_euler(op)
    dt = 50.0 * dt_exp
    s = O.rkl2_num_stages(dt, dt_exp)
    assert s == 14
    lam = _dct_lambda(32)
    U0 = sfft.dctn(u0, type=2, norm="ortho")
    u = u0.copy()
    for n in range(1, 11):
        u = O.rkl2_advance(lambda x: (op.M @ x.ravel()).reshape(x.shape), u, dt, s)
        if n in (1, 10):
            ref = sfft.idctn(U0 * _R(s, dt * lam) ** n, type=2, norm="ortho")
            err = np.linalg.norm(u - ref) / np.linalg.norm(ref)
            assert err < 1e-13, (n, err)


def test_be_pcg_config0_matches_dct_exact(heat):
    cfg, g, op = heat
    u0 = cfg["u"].numpy()
    dt = 50.0 * O.dt_euler(op)
    lam = _dct_lambda(32)
    U0 = sfft.dctn(u0, type=2, norm="ortho")
    u = u0.copy()
    iters = []
    for n in range(1, 11):
        u, k = O.be_pcg_solve(op, u, dt, rtol=1e-12)
        iters.append(k[0])
        ref = sfft.idctn(U0 / (1.0 - dt * lam) ** n, type=2, norm="ortho")
        err = np.linalg.norm(u - ref) / np.linalg.norm(ref)
        assert err < 1e-11, (n, err)
    assert all(0 < k < 200 for k in iters)


def _heat_kernel_1d(x, x0, sig2, L, nimg=4):
    out = 0.0
    for m in range(-nimg, nimg + 1):
        out = out + np.exp(-(x - x0 - 2 * m * L) ** 2 / (2 * sig2)) + np.exp(-(x + x0 - 2 * m * L) ** 2 / (2 * sig2))
    return out


def test_config0_converges_to_analytic_heat_kernel():
    """BASELINE configs[0]: the Gaussian bump (sigma = 4 cells) spreads like the
    continuum heat kernel (images for the zero-flux walls).  The gap is the
    O(h^2/sigma^2) spatial + time error; it must shrink with refinement."""
    errs = []
    for refine in (1, 2):
        n = 32 * refine
        h = 1.0 / refine
        g = W.uniform_cartesian(n, n, n, h)
        u0 = W.gaussian_bump(g, sigma=4.0, noise=0.0).numpy()
        op = O.Operator(g, [np.ones(g.shape)] * 3)
        dt_exp = O.dt_euler(op)
        t_end = 50.0 * (1.0 / 6.0) * 4          # fixed physical time
        nsteps = 4 * refine * refine             # dt/dt_exp fixed at 50 on both grids
        dt = t_end / nsteps
        s = O.rkl2_num_stages(dt, dt_exp)
        u = u0.copy()
        for _ in range(nsteps):
            u = O.rkl2_advance(lambda x: (op.M @ x.ravel()).reshape(x.shape), u, dt, s)
        sig2 = 16.0 + 2.0 * t_end
        xc = g.x1c
        k1 = _heat_kernel_1d(xc, 16.0, sig2, 32.0) * math.sqrt(16.0 / sig2)
        exact = k1[:, None, None] * k1[None, :, None] * k1[None, None, :]
        errs.append(np.linalg.norm(u - exact) / np.linalg.norm(exact))
    assert errs[0] < 5e-2 and errs[1] < 5e-3 and errs[1] < errs[0] / 3.0, errs


@pytest.mark.parametrize("method", ["rkl2", "be"])
def test_conservation_zero_flux(method):
    """Volume-weighted total is invariant under zero-flux walls (spherical, aniso)."""
    cfg = W.make_config("c1_spitzer64", shape=(10, 12, 16))
    g = cfg["grid"]
    T = cfg["T"].numpy()
    kap = O.spitzer_face_kappa(g, T, cfg["kappa0"], cfg["T_cut"])
    op = O.Operator(g, kap, cfg["b"].numpy())
    dt = 100.0 * O.dt_euler(op)
    tot0 = float(np.sum(op.WV * T.ravel()))
    if method == "rkl2":
        u = O.rkl2_advance(lambda x: (op.M @ x.ravel()).reshape(x.shape), T, dt,
                           O.rkl2_num_stages(dt, O.dt_euler(op)))
        tol = 1e-13
    else:
        u, _ = O.be_pcg_solve(op, T, dt, rtol=1e-12)
        tol = 1e-11
    assert abs(float(np.sum(op.WV * u.ravel())) - tot0) < tol * abs(tot0)
    assert np.max(np.abs(u - T)) > 1e-6 * np.max(T)   # something actually happened


def _tiny_aniso():
    cfg = W.make_config("c1_spitzer64", shape=(4, 5, 6))
    g = cfg["grid"]
    kap = O.spitzer_face_kappa(g, cfg["T"].numpy(), cfg["kappa0"], cfg["T_cut"])
    return cfg, g, O.Operator(g, kap, cfg["b"].numpy())


def test_pcg_matches_dense_direct_solve():
    cfg, g, op = _tiny_aniso()
    T = cfg["T"].numpy()
    for ratio in (1.0, 100.0, 1e4):
        dt = ratio * O.dt_euler(op)
        A = O.be_system(op, dt).toarray()
        x_direct = np.linalg.solve(A, op.WV * T.ravel())
        x, k = O.be_pcg_solve(op, T, dt, rtol=1e-14)
        # cond(A) ~ 2e6 here (cell volumes span 1e6): rtol 1e-14 -> ~1e-11 error
        assert np.linalg.norm(x.ravel() - x_direct) < 2e-11 * np.linalg.norm(x_direct), ratio
        assert k[0] <= 5 * g.ncells


def test_pcg_fig1_reading_z_kplus1():
    """DESIGN R8: Fig. 1 prints p_{k+1} = beta p_k + z_k; with z_k the method
    does not converge to the direct solution, with z_{k+1} it does."""
    cfg, g, op = _tiny_aniso()
    T = cfg["T"].numpy().ravel()
    dt = 100.0 * O.dt_euler(op)
    A = O.be_system(op, dt)
    b = op.WV * T
    x_direct = np.linalg.solve(A.toarray(), b)
    P = A.diagonal()
    x = T.copy()
    r = b - A @ x
    z = r / P
    p = z.copy()
    rr = r @ z
    for _ in range(g.ncells):
        y = A @ p
        al = rr / (p @ y)
        x = x + al * p
        r = r - al * y
        z_old = z
        z = r / P
        rold, rr = rr, r @ z
        p = (rr / rold) * p + z_old   # the printed index
    assert np.linalg.norm(x - x_direct) > 1e-6 * np.linalg.norm(x_direct)


def test_pcg_identity_and_zero_residual():
    cfg, g, op = _tiny_aniso()
    T = cfg["T"].numpy()
    x, k = O.be_pcg_solve(op, T, 0.0)            # A = diag(wV): Jacobi is exact
    assert k == [0] or k == [1]
    assert np.max(np.abs(x - T)) < 1e-15 * np.max(T)
    c = np.full(g.shape, 3.0)                    # L c = 0 -> r0 = 0 -> 0 iterations
    x, k = O.be_pcg_solve(op, c, 100.0 * O.dt_euler(op))
    assert k == [0] and np.array_equal(x, c)


def test_gershgorin_brute_force_and_bounds():
    cfg, g, op = _tiny_aniso()
    M = op.M.toarray()
    lam_g = np.max(np.abs(M).sum(axis=1))
    assert abs(O.dt_euler(op) - 2.0 / lam_g) < 1e-15 * 2.0 / lam_g
    rho = np.max(np.abs(np.linalg.eigvals(M)))
    assert lam_g >= rho * (1 - 1e-12)             # App. B theorem: a safe bound
    # App. B sqrt(p) tightness for symmetric matrices: uniform Cartesian (V const)
    for aniso in (False, True):
        gc = W.uniform_cartesian(6, 5, 7)
        rng = np.random.default_rng(5)
        kap = [rng.uniform(0.5, 2, gc.shape) for _ in range(3)]
        b = W.random_unit_b(gc, 2).numpy() if aniso else None
        opc = O.Operator(gc, kap, b)
        Mc = opc.M.toarray()
        assert np.max(np.abs(Mc - Mc.T)) < 1e-14 * np.max(np.abs(Mc))
        p = 27 if aniso else 7
        rho = np.max(np.abs(np.linalg.eigvalsh(Mc)))
        bound = 2.0 / O.dt_euler(opc)
        assert rho <= bound * (1 + 1e-12) and bound <= math.sqrt(p) * rho


def test_vector_field_componentwise():
    cfg = W.make_config("c2_visc64", shape=(6, 5, 8))
    g = cfg["grid"]
    op = O.Operator(g, [f.numpy() for f in cfg["visc_faces"]], None, cfg["rho"].numpy())
    v = cfg["v"].numpy()
    F = op.apply(v)
    for c in range(3):
        assert np.array_equal(F[c], op.apply(v[c]))
    dt = 500.0 * O.dt_euler(op)
    x, ks = O.be_pcg_solve(op, v, dt, rtol=1e-12)
    assert len(ks) == 3
    # weighted conservation: sum rho V v is invariant
    for c in range(3):
        t0 = np.sum(op.WV * v[c].ravel())
        assert abs(np.sum(op.WV * x[c].ravel()) - t0) < 1e-10 * np.sum(op.WV * np.abs(v[c].ravel()))


# ---------------------------------------------------------------- Sec. 3 / Sec. 6 properties
def _heat_op(shape=(15, 15, 15)):
    g = W.uniform_cartesian(*shape)
    return g, O.Operator(g, [np.ones(g.shape)] * 3)


@pytest.mark.parametrize("ratio", [5.0, 50.0, 500.0])
def test_rkl2_stable_and_nonnegative_on_config0_data(ratio):
    """PAPER.md:339 'strongly A-stable ... positive preserving', on BASELINE configs[0]
    data (Gaussian bump + noise): 20 super-steps keep the max-norm non-increasing and
    the solution non-negative (DESIGN R13: not for arbitrary data, see next test)."""
    cfg = W.make_config("c0_heat32", shape=(16, 16, 16))
    g = cfg["grid"]
    op = O.Operator(g, [f.numpy() for f in cfg["faces"]])
    dte = O.dt_euler(op)
    s = O.rkl2_num_stages(ratio * dte, dte)
    u = cfg["u"].numpy().copy()
    prev = np.abs(u).max()
    for _ in range(20):
        u = O.rkl2_advance(lambda x: (op.M @ x.ravel()).reshape(x.shape), u, ratio * dte, s)
        m = np.abs(u).max()
        assert m <= prev * (1 + 1e-13)
        assert u.min() >= -1e-12 * m
        prev = m


def test_rkl2_positivity_is_not_unconditional():
    """DESIGN R13: a single-cell delta goes negative after one RKL2 super-step once
    s > 2 (min ~ -2 % of the peak at 5 dt_Euler), while BE stays non-negative -- the
    'positive preserving' remark of PAPER.md:339 holds for smooth data only."""
    g, op = _heat_op()
    u0 = np.zeros(g.shape)
    u0[7, 7, 7] = 1.0
    dte = O.dt_euler(op)
    for ratio in (5.0, 50.0, 500.0):
        s = O.rkl2_num_stages(ratio * dte, dte)
        u = O.rkl2_advance(lambda x: (op.M @ x.ravel()).reshape(x.shape), u0, ratio * dte, s)
        ub, _ = O.be_pcg_solve(op, u0, ratio * dte, rtol=1e-13)
        assert u.min() < -1e-3
        assert ub.min() >= -1e-12
        assert abs(u.sum() - 1.0) < 1e-12 and abs(ub.sum() - 1.0) < 1e-9   # both conserve


def test_be_first_order_in_time():
    """BE (Eq. 4) is first order: on u' = lam u the error at fixed T halves with dt."""
    lam = -np.logspace(-1, 1, 20)
    T = 0.5
    errs = []
    for n in (16, 32, 64):
        dt = T / n
        u = np.ones_like(lam)
        for _ in range(n):
            u = u / (1.0 - dt * lam)
        errs.append(np.linalg.norm(u - np.exp(lam * T)))
    order = math.log2(errs[1] / errs[2])
    assert 0.8 < order < 1.2, errs


def test_fig3_speedup_model():
    """PAPER.md:149 (Fig. 3): RKL2 vs explicit Euler speedup = ratio / s, one sub-step
    costing one Euler step; s from Eq. (5) makes the curve jagged: between jumps of s
    it grows strictly with the ratio."""
    sp = lambda r: r / O.rkl2_num_stages(r, 1.0)  # noqa: E731
    assert sp(1.0) == 0.5 and sp(100.0) == 5.0 and abs(sp(500.0) - 500.0 / 45.0) < 1e-12
    rs = np.linspace(1.0, 300.0, 3000)
    ss = [O.rkl2_num_stages(r, 1.0) for r in rs]
    for a in range(len(rs) - 1):
        if ss[a] == ss[a + 1]:
            assert sp(rs[a + 1]) > sp(rs[a])
        else:
            assert ss[a + 1] == ss[a] + 1


def test_rkl2_and_be_agree_on_lagged_conduction():
    """PAPER.md Sec. 6 validation (Fig. 10): with lagged Spitzer diffusivity both
    methods advance the same nonlinear problem -- 5 steps at 20 dt_Euler differ by a
    few per cent at most."""
    cfg = W.make_config("c1_spitzer64", shape=(12, 10, 40))
    g = cfg["grid"]
    b = cfg["b"].numpy()
    Tr = cfg["T"].numpy().copy()
    Tb = Tr.copy()
    dt = None
    for _ in range(5):
        opr = O.Operator(g, O.spitzer_face_kappa(g, Tr, cfg["kappa0"], cfg["T_cut"]), b)
        opb = O.Operator(g, O.spitzer_face_kappa(g, Tb, cfg["kappa0"], cfg["T_cut"]), b)
        if dt is None:
            dt = 20.0 * O.dt_euler(opr)
        s = O.rkl2_num_stages(dt, O.dt_euler(opr))
        Tr = O.rkl2_advance(lambda x: (opr.M @ x.ravel()).reshape(x.shape), Tr, dt, s)
        Tb, _ = O.be_pcg_solve(opb, Tb, dt, rtol=1e-12)
    d = np.linalg.norm(Tr - Tb) / np.linalg.norm(Tb)
    assert d < 0.05
