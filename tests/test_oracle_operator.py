"""Pins for the oracle's geometry, lagged diffusivity and operator F(u).

Independent checks: closed-form volumes/areas, the DCT/FFT eigen-decomposition
of the constant-coefficient Laplacian (scipy.fft), brute-force central
differences of the discrete energy, conservation / symmetry / semi-definiteness
invariants, and second-order convergence to div(kappa b b.grad u) computed
symbolically (sympy) for manufactured solutions.
"""
import math

import numpy as np
import pytest
import scipy.fft as sfft
import sympy as sy

import workloads as W
from oracle import core as O


def _rand_faces(grid, rng, lo=0.5, hi=2.0):
    return [rng.uniform(lo, hi, grid.shape) for _ in range(3)]


def _rand_b(grid, rng):
    v = rng.normal(size=(3,) + grid.shape)
    return v / np.sqrt((v * v).sum(0))


# ------------------------------------------------------------------ geometry
def test_sphere_volume_and_area_closed_form():
    g = W.spherical_grid(12, 9, 16, r0=1.0, r1=3.0, dr0=0.05)
    geo = O.geometry(g)
    assert abs(geo["V"].sum() - 4 * math.pi / 3 * (27 - 1)) < 1e-12 * 4 * math.pi * 9
    i = 5
    area = geo["A"][0][i].sum()
    assert abs(area - 4 * math.pi * g.x1f[i + 1] ** 2) < 1e-12 * area


def test_geometric_faces_first_cell_and_ratio():
    f = W.geometric_faces(1.0, 20.0, 64, 0.005)
    d = np.diff(f)
    assert abs(d[0] - 0.005) < 1e-12 and abs(f[-1] - 20.0) < 1e-12
    q = d[1:] / d[:-1]
    assert np.ptp(q[:-1]) < 1e-9


# ------------------------------------------------------------------ kappa
def test_spitzer_kappa_closed_form():
    g = W.uniform_cartesian(3, 1, 1)
    Tc, k0 = 5.0e5, 2.0
    for T, expect in [(Tc, k0 * Tc ** 2.5), (2 * Tc, k0 * (2 * Tc) ** 2.5),
                      (Tc / 2, k0 * Tc ** 2.5 * 2.0 ** -5)]:
        k = O.spitzer_face_kappa(g, np.full(g.shape, T), k0, Tc)
        assert abs(k[0][0, 0, 0] - expect) < 1e-13 * expect
        assert k[0][2, 0, 0] == 0.0 and k[1].max() == 0.0  # no + neighbour
    # face temperature is the mean of the two cells
    T = np.array([1.0e6, 3.0e6, 3.0e6]).reshape(3, 1, 1)
    k = O.spitzer_face_kappa(g, T, 1.0, Tc)
    assert abs(k[0][0, 0, 0] - (2.0e6) ** 2.5) < 1e-13 * 2.0e6 ** 2.5
    # beta cut-off is continuous at T_cut
    assert abs(O.beta_tcut(Tc * (1 - 1e-12), Tc) - 1.0) < 1e-11


# tanh(1), written out (not computed): 0.76159415595576488812 (Abramowitz & Stegun Table 4.11)
TANH1 = 0.7615941559557649


def test_fc_profile_hand_values():
    """PAPER.md:183 f_c(r) = 0.5 (1 - tanh[(r - 10 R_sun) / 0.5 R_sun]) at hand-evaluated
    points: the half-value radius, one width either side, far inside / outside, the
    f_c + f_nc = 1 symmetry about 10 R_sun, monotone decrease, and f_c = 1 when off."""
    f = lambda r: float(O.f_c(np.array([r]), 10.0, 0.5)[0])  # noqa: E731
    assert f(10.0) == 0.5
    assert abs(f(10.5) - 0.5 * (1.0 - TANH1)) <= 1e-16
    assert abs(f(9.5) - 0.5 * (1.0 + TANH1)) <= 1e-16
    # the logistic form 0.5 (1 - tanh x) = 1 / (1 + e^{2x}), x = (r - 10)/0.5, far from the
    # half-value radius (r << 10: f_c -> 1, e^{-36} below 1 at r = 1; r >> 10: f_c -> 0)
    for r, x in ((1.0, -18.0), (8.0, -4.0), (12.0, 4.0), (15.0, 10.0), (19.5, 19.0)):
        assert abs(f(r) - 1.0 / (1.0 + math.exp(2.0 * x))) <= 1e-12 * f(r) + 4.5e-16, r
    r = np.linspace(1.0, 20.0, 2001)
    fc = O.f_c(r, 10.0, 0.5)
    assert np.all(np.diff(fc) <= 0.0)
    np.testing.assert_allclose(O.f_c(10.0 + (r - 1.0), 10.0, 0.5) + O.f_c(10.0 - (r - 1.0), 10.0, 0.5), 1.0,
                               rtol=0, atol=2e-16)
    assert np.all(O.f_c(r, 10.0, 0.0) == 1.0)


def test_fc_face_kappa_evaluation_radius():
    """The f_c factor of the lagged face diffusivity (PAPER.md:173 boxed term) is taken at
    the face's own radius: r_{i+1/2} for r-faces, the cell centre r_i for theta / phi faces
    (DESIGN R3).  A grid with an r-face exactly at 10 R_sun and a cell centred at 10.5."""
    x1f = np.array([9.0, 9.5, 10.0, 11.0, 12.0])      # centres 9.25, 9.75, 10.5, 11.5
    g = W.Grid("spherical", x1f, np.linspace(0.5, 2.5, 4), np.linspace(0.0, 1.0, 4), False)
    T = np.full(g.shape, 1.0e6)
    on = O.spitzer_face_kappa(g, T, 1.0, 5e5, 10.0, 0.5)
    off = O.spitzer_face_kappa(g, T, 1.0, 5e5, 10.0, 0.0)
    assert on[0][1, 0, 0] == 0.5 * off[0][1, 0, 0]                             # r-face at r = 10
    assert abs(on[1][2, 0, 0] / off[1][2, 0, 0] - 0.5 * (1 - TANH1)) <= 1e-15  # theta face, r_c = 10.5
    assert abs(on[2][2, 1, 0] / off[2][2, 1, 0] - 0.5 * (1 - TANH1)) <= 1e-15  # phi face, r_c = 10.5
    assert abs(on[0][0, 0, 0] / off[0][0, 0, 0] - 0.5 * (1 + TANH1)) <= 1e-15  # r-face at 9.5


# ------------------------------------------------------------------ spectral pin
@pytest.mark.parametrize("shape,h,periodic", [((6, 7, 8), (1.0, 0.5, 2.0), False),
                                              ((5, 4, 9), (0.3, 0.3, 0.7), True)])
def test_isotropic_cartesian_matches_dct_eigendecomposition(shape, h, periodic, rng):
    n1, n2, n3 = shape
    g = W.Grid("cartesian", np.arange(n1 + 1) * h[0], np.arange(n2 + 1) * h[1],
               np.arange(n3 + 1) * h[2], periodic3=periodic)
    kap = 1.7
    u = rng.normal(size=shape)
    F = O.op_apply(g, u, [np.full(shape, kap)] * 3)
    U = sfft.dctn(u, type=2, norm="ortho", axes=(0, 1))
    lam1 = -(4 / h[0] ** 2) * np.sin(np.pi * np.arange(n1) / (2 * n1)) ** 2
    lam2 = -(4 / h[1] ** 2) * np.sin(np.pi * np.arange(n2) / (2 * n2)) ** 2
    if periodic:
        U = np.fft.fft(U, axis=2)
        lam3 = -(4 / h[2] ** 2) * np.sin(np.pi * np.arange(n3) / n3) ** 2
    else:
        U = sfft.dct(U, type=2, norm="ortho", axis=2)
        lam3 = -(4 / h[2] ** 2) * np.sin(np.pi * np.arange(n3) / (2 * n3)) ** 2
    lam = lam1[:, None, None] + lam2[None, :, None] + lam3[None, None, :]
    X = kap * lam * U
    if periodic:
        X = np.real(np.fft.ifft(X, axis=2))
    else:
        X = sfft.idct(X, type=2, norm="ortho", axis=2)
    ref = sfft.idctn(X, type=2, norm="ortho", axes=(0, 1))
    assert np.max(np.abs(F - ref)) < 1e-12 * np.max(np.abs(ref))


# ------------------------------------------------------------------ energy brute force
SHAPES = [((1, 1, 1), False), ((1, 3, 4), False), ((3, 1, 2), True), ((2, 2, 1), True),
          ((2, 2, 2), True), ((3, 4, 5), False), ((4, 3, 6), True)]


@pytest.mark.parametrize("shape,periodic", SHAPES)
@pytest.mark.parametrize("aniso", [False, True])
def test_operator_is_minus_energy_gradient(shape, periodic, aniso, rng):
    n1, n2, n3 = shape
    g = W.Grid("spherical", 1.0 + np.cumsum(np.r_[0, rng.uniform(0.1, 0.3, n1)]),
               np.linspace(0.4, 2.5, n2 + 1),
               np.linspace(0.0, 2 * math.pi if periodic else 1.0, n3 + 1), periodic3=periodic)
    kap = _rand_faces(g, rng)
    b = _rand_b(g, rng) if aniso else None
    u = rng.normal(size=shape)
    Lu = O.assemble_L(g, kap, b) @ u.ravel()
    grad = np.zeros(g.ncells)
    for i in range(g.ncells):
        e = np.zeros(g.ncells)
        e[i] = 1.0
        grad[i] = 0.5 * (O.energy(g, u.ravel() + e, kap, b) - O.energy(g, u.ravel() - e, kap, b))
    scale = max(1.0, np.max(np.abs(Lu)))
    assert np.max(np.abs(Lu + grad)) < 1e-10 * scale


@pytest.mark.parametrize("aniso", [False, True])
def test_symmetric_conservative_semidefinite(aniso, rng):
    g = W.spherical_grid(5, 6, 7, r0=1.0, r1=2.0, dr0=0.1)
    kap = _rand_faces(g, rng)
    b = _rand_b(g, rng) if aniso else None
    L = O.assemble_L(g, kap, b).toarray()
    s = np.max(np.abs(L))
    assert np.max(np.abs(L - L.T)) < 1e-14 * s
    assert np.max(np.abs(L.sum(axis=0))) < 1e-13 * s          # sum_i (L u)_i = 0
    ev = np.linalg.eigvalsh(L)
    assert ev.max() < 1e-12 * s                                 # -L >= 0
    assert abs(np.linalg.eigvalsh(L)[-1]) < 1e-12 * s           # constants in the null space
    nnz = (np.abs(L) > 0).sum(axis=1).reshape(g.shape)
    assert nnz[2, 2, 3] == (27 if aniso else 7)


# ------------------------------------------------------------------ manufactured solutions
X, Y, Z = sy.symbols("x y z", real=True)


def _lambdify(expr):
    f = sy.lambdify((X, Y, Z), expr, "numpy")
    return lambda x, y, z: np.broadcast_to(np.asarray(f(x, y, z), dtype=np.float64), np.broadcast(x, y, z).shape)


def _manufactured(kind):
    u = sy.sin(1.3 * X + 0.4) * sy.cos(0.9 * Y - 0.2) * sy.exp(0.5 * Z)
    kap = 1.0 + 0.3 * X * X + 0.2 * sy.sin(Y + Z)
    if kind == "iso":
        F = sum(sy.diff(kap * sy.diff(u, v), v) for v in (X, Y, Z))
        return u, kap, None, F
    if kind == "const_b":
        bvec = sy.Matrix([1, 2, 2]) / 3
    else:  # dipole direction, tilted
        m = sy.Matrix([sy.Rational(1, 2), 0, sy.sqrt(3) / 2])
        rv = sy.Matrix([X, Y, Z])
        rr = sy.sqrt(X * X + Y * Y + Z * Z)
        B = (3 * (m.dot(rv)) * rv / rr ** 2 - m) / rr ** 3
        bvec = B / sy.sqrt(B.dot(B))
    grad = sy.Matrix([sy.diff(u, v) for v in (X, Y, Z)])
    q = kap * bvec * bvec.dot(grad)
    F = sum(sy.diff(q[d], v) for d, v in enumerate((X, Y, Z)))
    return u, kap, bvec, F


def _sph_patch(n):
    return W.Grid("spherical", np.linspace(1.0, 1.5, n + 1), np.linspace(0.6, 1.2, n + 1),
                  np.linspace(0.3, 0.9, n + 1), periodic3=False)


def _eval_on(grid, fx, where):
    """Evaluate a Cartesian function at cell centres ('c') or at the + faces of
    direction d (where = d)."""
    r = grid.x1c[:, None, None]
    t = grid.x2c[None, :, None]
    p = grid.x3c[None, None, :]
    if where == 0:
        r = np.append(grid.x1f[1:-1], np.nan)[:, None, None]
    elif where == 1:
        t = np.append(grid.x2f[1:-1], np.nan)[None, :, None]
    elif where == 2:
        p = np.append(grid.x3f[1:-1], np.nan)[None, None, :]
    x = r * np.sin(t) * np.cos(p)
    y = r * np.sin(t) * np.sin(p)
    z = r * np.cos(t) + 0 * p
    return np.nan_to_num(fx(x, y, z))


@pytest.mark.parametrize("kind", ["iso", "const_b", "dipole_b"])
def test_second_order_convergence_to_continuum(kind):
    u_e, kap_e, b_e, F_e = _manufactured(kind)
    fu, fk, fF = _lambdify(u_e), _lambdify(kap_e), _lambdify(F_e)
    errs = []
    ns = (16, 32, 48)
    for n in ns:
        g = _sph_patch(n)
        u = _eval_on(g, fu, "c")
        kap = [_eval_on(g, fk, d) for d in range(3)]
        b = None
        if b_e is not None:
            bx, by, bz = [_eval_on(g, _lambdify(b_e[d]), "c") for d in range(3)]
            t = g.x2c[None, :, None]
            p = g.x3c[None, None, :]
            br = bx * np.sin(t) * np.cos(p) + by * np.sin(t) * np.sin(p) + bz * np.cos(t)
            bt = bx * np.cos(t) * np.cos(p) + by * np.cos(t) * np.sin(p) - bz * np.sin(t)
            bp = -bx * np.sin(p) + by * np.cos(p)
            b = [br, bt, bp]
        F = O.op_apply(g, u, kap, b)
        Fx = _eval_on(g, fF, "c")
        inner = (slice(2, -2),) * 3
        e = F[inner] - Fx[inner]
        errs.append(math.sqrt(np.mean(e * e) / np.mean(Fx[inner] ** 2)))
    o1 = math.log(errs[0] / errs[1]) / math.log(ns[1] / ns[0])
    o2 = math.log(errs[1] / errs[2]) / math.log(ns[2] / ns[1])
    assert errs[2] < 1e-3 and o2 > 1.8 and o1 > 1.6, (errs, o1, o2)
