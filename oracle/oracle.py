"""ORACLE — test infrastructure, NOT part of the product.

Plain, slow, obviously-correct CPU reference (numpy/scipy, float64) of the hot
path of Caplan et al., "Advancing parabolic operators in thermodynamic MHD
models: explicit super time-stepping versus implicit schemes with Krylov
solvers" (arxiv 1610.01265; /root/reference/PAPER.md).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module.  It shares no code with the CUDA path
(paper_1610_01265_b200/) and never imports it.

Structure (each function cites the passage it follows; "PAPER.md:L" is a line
of /root/reference/PAPER.md, DESIGN.md "R<n>" is a listed reading):
  geometry()            cell volumes, face areas / centre distances    PAPER.md:193 (Sec. 4.2), DESIGN R1
  spitzer_face_kappa()  lagged kappa0*beta_Tcut(T)*T^(5/2) at faces     PAPER.md:33, :173, :187, DESIGN R3
  assemble_L()          symmetric operator from the discrete energy     PAPER.md:173 / :181 boxed terms, DESIGN R2
  energy()              the same quadratic form evaluated directly      DESIGN R2
  op_apply()            F(u) = L u / (w V)                              PAPER.md:25 Eq. (1)
  dt_euler()            Gershgorin bound, dt = 2/max row sum |M|       PAPER.md:512-538 (App. B)
  rkl2_num_stages()     s = ceil((sqrt(9+16 dt/dt_exp)-1)/2), s>=2     PAPER.md:142 Eq. (5), DESIGN R5
  rkl2_coeffs()         b_j, mu_j, nu_j, mu~_j, gamma~_j               PAPER.md:134-138, DESIGN R6
  rkl2_advance()        Fig. 2 recursion                               PAPER.md:117-125 (Fig. 2)
  rkl2_hybrid_advance() Euler prefix + RKL2 sub-cycling               PAPER.md:341 (Sec. 6)
  be_system()           A = wV - dt L (symmetric form of Eq. 4)        PAPER.md:45-60 Eqs. (2)-(4), DESIGN R7
  pcg()                 Fig. 1 PCG, point-Jacobi PC1                   PAPER.md:70-92 (Fig. 1), :468-470 (App. A), DESIGN R8
  be_pcg_solve()        BE step via pcg() per component

Every function is pinned by `-m "not gpu"` tests in tests/test_oracle_*.py
(closed forms, DCT-exact discrete solutions, brute force, conservation,
manufactured-solution convergence, paper-printed values).  No function is
"parity unpinned".
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp

# --------------------------------------------------------------------------
# index helpers
# --------------------------------------------------------------------------


def _plus(arr, d, periodic3):
    """arr evaluated at cell + e_d (entries with no +1 neighbour are garbage
    and must be masked with _valid)."""
    if d == 2 and periodic3:
        return np.roll(arr, -1, axis=2)
    out = np.array(arr, copy=True)
    src = [slice(None)] * 3
    dst = [slice(None)] * 3
    src[d] = slice(1, None)
    dst[d] = slice(0, -1)
    out[tuple(dst)] = arr[tuple(src)]
    return out


def _valid(shape, d, periodic3):
    """True where cell + e_d exists (a face in direction d on the + side)."""
    m = np.ones(shape, dtype=bool)
    if d == 2 and periodic3:
        return m
    sl = [slice(None)] * 3
    sl[d] = slice(shape[d] - 1, None)
    m[tuple(sl)] = False
    return m


# --------------------------------------------------------------------------
# geometry  (Sec. 4.2: logically rectangular non-uniform
# spherical grid; DESIGN R1: finite-volume metrics of that grid)
# --------------------------------------------------------------------------


def geometry(grid):
    """Return dict with V (cell volumes) and, per direction d, A[d] (area of
    the + face) and H[d] (distance between the centres the + face separates).

    Spherical (r, theta, phi):
      V  = (r+^3 - r-^3)/3 * (cos th- - cos th+) * dphi
      r-face  : A = r_{i+1/2}^2 (cos th- - cos th+) dphi,   h = r_{i+1} - r_i
      th-face : A = (r+^2 - r-^2)/2 sin th_{j+1/2} dphi,    h = r_i (th_{j+1} - th_j)
      ph-face : A = (r+^2 - r-^2)/2 (th+ - th-),            h = r_i sin th_j (ph_{k+1} - ph_k)
    Cartesian: V = dx dy dz, A = product of the two transverse widths,
      h = centre spacing.
    """
    n1, n2, n3 = grid.shape
    x1f, x2f, x3f = grid.x1f, grid.x2f, grid.x3f
    x1c, x2c, x3c = grid.x1c, grid.x2c, grid.x3c
    d1, d2, d3 = np.diff(x1f), np.diff(x2f), np.diff(x3f)
    # centre spacing towards +1 neighbour (garbage at the last index unless periodic)
    c1 = np.append(x1c[1:] - x1c[:-1], np.nan)
    c2 = np.append(x2c[1:] - x2c[:-1], np.nan)
    if grid.periodic3:
        c3 = np.append(x3c[1:] - x3c[:-1], x3c[0] + grid.period3 - x3c[-1])
    else:
        c3 = np.append(x3c[1:] - x3c[:-1], np.nan)
    I = (slice(None), None, None)
    J = (None, slice(None), None)
    K = (None, None, slice(None))
    shape = (n1, n2, n3)
    with np.errstate(invalid="ignore"):
        if grid.geom == "spherical":
            r3 = (x1f[1:] ** 3 - x1f[:-1] ** 3) / 3.0
            r2 = (x1f[1:] ** 2 - x1f[:-1] ** 2) / 2.0
            mu = np.cos(x2f[:-1]) - np.cos(x2f[1:])
            V = r3[I] * mu[J] * d3[K]
            A1 = (x1f[1:] ** 2)[I] * mu[J] * d3[K]
            H1 = c1[I] + 0 * mu[J] * d3[K]
            A2 = r2[I] * np.sin(x2f[1:])[J] * d3[K]
            H2 = x1c[I] * c2[J] + 0 * d3[K]
            A3 = r2[I] * d2[J] + 0 * d3[K]
            H3 = x1c[I] * np.sin(x2c)[J] * c3[K]
        elif grid.geom == "cartesian":
            V = d1[I] * d2[J] * d3[K]
            A1 = 0 * d1[I] + d2[J] * d3[K]
            H1 = c1[I] + 0 * d2[J] * d3[K]
            A2 = d1[I] * d3[K] + 0 * d2[J]
            H2 = c2[J] + 0 * d1[I] * d3[K]
            A3 = d1[I] * d2[J] + 0 * d3[K]
            H3 = c3[K] + 0 * d1[I] * d2[J]
        else:
            raise ValueError(grid.geom)
    A = [np.broadcast_to(a, shape).copy() for a in (A1, A2, A3)]
    H = [np.broadcast_to(h, shape).copy() for h in (H1, H2, H3)]
    for d in range(3):
        m = _valid(shape, d, grid.periodic3)
        A[d][~m] = 0.0
        H[d][~m] = np.nan
    return {"V": np.broadcast_to(V, shape).copy(), "A": A, "H": H}


# --------------------------------------------------------------------------
# lagged Spitzer diffusivity (PAPER.md:33 lagged diffusivity; :173 boxed term
# beta_Tcut(T) f_c(r) kappa0 T^(5/2); :187 beta_Tcut; DESIGN R3 face average)
# --------------------------------------------------------------------------


def beta_tcut(T, T_cut):
    """beta = (T/T_cut)^(5/2) for T < T_cut, else 1 (T_cut<=0: off)."""
    T = np.asarray(T, dtype=np.float64)
    if T_cut <= 0:
        return np.ones_like(T)
    return np.where(T < T_cut, (T / T_cut) ** 2.5, 1.0)


def f_c(r, fc_r0, fc_w):
    """f_c(r) = 0.5 (1 - tanh((r - 10)/0.5)); fc_w <= 0 disables (=1)."""
    if fc_w <= 0:
        return np.ones_like(np.asarray(r, dtype=np.float64))
    return 0.5 * (1.0 - np.tanh((np.asarray(r) - fc_r0) / fc_w))


def spitzer_face_kappa(grid, T, kappa0, T_cut, fc_r0=10.0, fc_w=0.0):
    """Face diffusivity kappa_f = kappa0 f_c(r_f) beta(Tf) Tf^(5/2), Tf = mean of
    the two adjacent cell temperatures (DESIGN R3).  Faces without a + neighbour
    are 0 (zero-flux boundary).  Returns [k1, k2, k3] in the + face convention."""
    T = np.asarray(T, dtype=np.float64)
    n1, n2, n3 = grid.shape
    out = []
    for d in range(3):
        Tf = 0.5 * (T + _plus(T, d, grid.periodic3))
        k = kappa0 * beta_tcut(Tf, T_cut) * Tf ** 2.5
        if grid.geom == "spherical" and fc_w > 0:
            rf = grid.x1f[1:] if d == 0 else grid.x1c
            k = k * f_c(rf, fc_r0, fc_w)[:, None, None]
        k = np.where(_valid(grid.shape, d, grid.periodic3), k, 0.0)
        out.append(np.ascontiguousarray(k))
    return out


# --------------------------------------------------------------------------
# the operator  (DESIGN R2: discrete energy -> symmetric conservative L)
# --------------------------------------------------------------------------


def _face_coeffs(grid, geo, kappa):
    """Isotropic face coefficient K_f = kappa_f A_f / h_f per direction."""
    K = []
    for d in range(3):
        m = _valid(grid.shape, d, grid.periodic3)
        with np.errstate(invalid="ignore", divide="ignore"):
            Kd = np.asarray(kappa[d], dtype=np.float64) * geo["A"][d] / geo["H"][d]
        K.append(np.where(m, Kd, 0.0))
    return K


def _vertex_data(grid, geo, kappa, b):
    """Vertices (i+1/2, j+1/2, k+1/2) surrounded by 8 existing cells
    c_s = base + s, s in {0,1}^3 (periodic wrap in dim 3).  DESIGN R2:
      g_a   = 1/4 sum_{s: s_a=0} (u(c_{s+e_a}) - u(c_s)) / h_a(c_s)
      b_v   = 1/8 sum_s b(c_s)            (component-wise mean, not renormalised)
      kap_v = 1/12 sum of the 12 faces around the vertex (4 per direction)
      V_v   = 1/8 sum_s V(c_s)
      E_v   = 1/2 V_v kap_v (b_v . g_v)^2
    Returns (ids[8], C = V_v kap_v, wts[8]) on the vertex mask, where
    wts_p = b_v . d(g_v)/du_p so that E_v = 1/2 C (sum_p wts_p u_p)^2."""
    p3 = grid.periodic3
    shape = grid.shape
    m = _valid(shape, 0, p3) & _valid(shape, 1, p3) & _valid(shape, 2, p3)

    def at(arr, s):
        out = arr
        for d in range(3):
            if s[d]:
                out = _plus(out, d, p3)
        return out

    octs = [(s0, s1, s2) for s0 in (0, 1) for s1 in (0, 1) for s2 in (0, 1)]
    idx = np.arange(grid.ncells).reshape(shape)
    ids = [at(idx, s)[m] for s in octs]
    V = geo["V"]
    Vv = sum(at(V, s) for s in octs)[m] / 8.0
    bv = [sum(at(np.asarray(b[a], dtype=np.float64), s) for s in octs)[m] / 8.0 for a in range(3)]
    kv = 0.0
    for a in range(3):
        ka = np.asarray(kappa[a], dtype=np.float64)
        kv = kv + sum(at(ka, s) for s in octs if s[a] == 0)[m]
    kv = kv / 12.0
    wts = [np.zeros(int(m.sum())) for _ in octs]
    for a in range(3):
        Ha = geo["H"][a]
        for p, s in enumerate(octs):
            if s[a] == 0:
                hs = at(Ha, s)[m]
                q = octs.index(tuple(1 if d == a else s[d] for d in range(3)))
                wts[p] = wts[p] - bv[a] * 0.25 / hs
                wts[q] = wts[q] + bv[a] * 0.25 / hs
    return ids, Vv * kv, wts


def assemble_L(grid, kappa, b=None, geo=None):
    """Sparse symmetric L with (L u)_i = -dE/du_i  (DESIGN R2).

    Isotropic (b None; PAPER.md:181 viscosity term div(nu rho grad v), :329 the
    constant-coefficient heat test):   E = 1/2 sum_faces K_f (u_R - u_L)^2.
    Anisotropic (PAPER.md:173 boxed term div(kappa b b.grad T)):
                                       E = 1/2 sum_vertices V_v kap_v (b_v.g_v)^2.
    The continuum limit of -dE/du / V is div(kappa grad u), resp.
    div(kappa b b.grad u).  Symmetric and conservative by construction.
    """
    geo = geometry(grid) if geo is None else geo
    n = grid.ncells
    rows, cols, vals = [], [], []
    idx = np.arange(n).reshape(grid.shape)
    if b is None:
        K = _face_coeffs(grid, geo, kappa)
        for d in range(3):
            m = _valid(grid.shape, d, grid.periodic3)
            L_ = idx[m]
            R_ = _plus(idx, d, grid.periodic3)[m]
            k = K[d][m]
            # E_f = 1/2 k (uR - uL)^2  ->  Hessian [[k,-k],[-k,k]],  L = -Hessian
            rows += [L_, R_, L_, R_]
            cols += [L_, R_, R_, L_]
            vals += [-k, -k, k, k]
    else:
        ids, C, wts = _vertex_data(grid, geo, kappa, b)
        # E_v = 1/2 C (w.u)^2 -> Hessian_pq = C w_p w_q,  L = -Hessian
        for p in range(8):
            for q in range(8):
                rows.append(ids[p])
                cols.append(ids[q])
                vals.append(-C * wts[p] * wts[q])
    if not rows:
        return sp.csr_matrix((n, n))
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    vals = np.concatenate(vals)
    return sp.csr_matrix((vals, (rows, cols)), shape=(n, n))


def energy(grid, u, kappa, b=None, geo=None):
    """E(u) of DESIGN R2 evaluated directly from u (no matrix)."""
    geo = geometry(grid) if geo is None else geo
    u = np.asarray(u, dtype=np.float64).reshape(grid.shape)
    E = 0.0
    if b is None:
        K = _face_coeffs(grid, geo, kappa)
        for d in range(3):
            m = _valid(grid.shape, d, grid.periodic3)
            du = (_plus(u, d, grid.periodic3) - u)[m]
            E += 0.5 * float(np.sum(K[d][m] * du * du))
    else:
        uf = u.ravel()
        ids, C, wts = _vertex_data(grid, geo, kappa, b)
        bg = sum(wts[p] * uf[ids[p]] for p in range(8))
        E += 0.5 * float(np.sum(C * bg * bg))
    return E


class Operator:
    """F(u) = L u / (w V) (Eq. 1), M = diag(1/(wV)) L (Eq. 3)."""

    def __init__(self, grid, kappa, b=None, w=None):
        self.grid = grid
        self.geo = geometry(grid)
        self.L = assemble_L(grid, kappa, b, self.geo)
        wv = self.geo["V"] if w is None else np.asarray(w, dtype=np.float64) * self.geo["V"]
        self.WV = np.ascontiguousarray(wv).ravel()
        self.M = sp.diags(1.0 / self.WV) @ self.L
        self.M = sp.csr_matrix(self.M)

    def apply(self, u):
        """F(u) for u of shape grid.shape or (ncomp,)+grid.shape (component-wise)."""
        u = np.asarray(u, dtype=np.float64)
        if u.ndim == 4:
            return np.stack([self.apply(x) for x in u])
        return (self.L @ u.ravel() / self.WV).reshape(self.grid.shape)


def op_apply(grid, u, kappa, b=None, w=None):
    return Operator(grid, kappa, b, w).apply(u)


# --------------------------------------------------------------------------
# Appendix B: Gershgorin estimate of the explicit Euler limit
# --------------------------------------------------------------------------


def dt_euler(op: Operator) -> float:
    """PAPER.md:512 dt_Euler = 2/|lambda|_max with PAPER.md:536
    |lambda|_max <= max_j sum_i |M_ji| (absolute row sums of M)."""
    rs = np.asarray(abs(op.M).sum(axis=1)).ravel()
    lam = float(rs.max()) if rs.size else 0.0
    return math.inf if lam == 0.0 else 2.0 / lam


# --------------------------------------------------------------------------
# RKL2 super time-stepping (Sec. 3, Fig. 2, Eq. 5)
# --------------------------------------------------------------------------


def rkl2_num_stages(dt, dt_exp, force_odd=False):
    """PAPER.md:142 Eq. (5) in BASELINE north_star form
    s = ceil((sqrt(9 + 16 dt/dt_exp) - 1)/2), floored at 2 (DESIGN R5)."""
    ratio = dt / dt_exp
    s = int(math.ceil((math.sqrt(9.0 + 16.0 * ratio) - 1.0) / 2.0))
    s = max(s, 2)
    if force_odd and s % 2 == 0:  # PAPER.md:144 "ensuring s is odd"
        s += 1
    return s


def rkl2_coeffs(s):
    """PAPER.md:134-138.  Arrays indexed by stage j = 0..s (index 0 unused):
    b_j, mu_j, nu_j, mut_j (mu~), gt_j (gamma~ = (b_{j-1} - 1) mu~_j, DESIGN R6)."""
    b = np.zeros(s + 1)
    for j in range(s + 1):
        b[j] = 1.0 / 3.0 if j <= 2 else (j * j + j - 2.0) / (2.0 * j * (j + 1.0))
    w1 = 4.0 / (s * s + s - 2.0)
    mu = np.zeros(s + 1)
    nu = np.zeros(s + 1)
    mut = np.zeros(s + 1)
    gt = np.zeros(s + 1)
    mut[1] = 4.0 / (3.0 * (s * s + s - 2.0))  # = b_1 w1
    for j in range(2, s + 1):
        mu[j] = (2.0 * j - 1.0) / j * b[j] / b[j - 1]
        nu[j] = -(j - 1.0) / j * b[j] / b[j - 2]
        mut[j] = 4.0 * (2.0 * j - 1.0) / (j * (s * s + s - 2.0)) * b[j] / b[j - 1]
        gt[j] = (b[j - 1] - 1.0) * mut[j]
    return {"b": b, "mu": mu, "nu": nu, "mut": mut, "gt": gt, "w1": w1}


def rkl2_advance(apply_M, u0, dt, s):
    """PAPER.md:117-125 (Fig. 2) / BASELINE north_star:
      M0 = M u^n;  Y1 = u^n + mu~_1 dt M0
      Y_j = mu_j Y_{j-1} + nu_j Y_{j-2} + (1-mu_j-nu_j) u^n
            + mu~_j dt M Y_{j-1} + gamma~_j dt M0,   j = 2..s
      u^{n+1} = Y_s
    apply_M: callable u -> M u (any shape)."""
    c = rkl2_coeffs(s)
    y0 = np.array(u0, dtype=np.float64)
    M0 = apply_M(y0)
    ym2 = y0
    ym1 = y0 + c["mut"][1] * dt * M0
    for j in range(2, s + 1):
        yj = (c["mu"][j] * ym1 + c["nu"][j] * ym2 + (1.0 - c["mu"][j] - c["nu"][j]) * y0
              + c["mut"][j] * dt * apply_M(ym1) + c["gt"][j] * dt * M0)
        ym2, ym1 = ym1, yj
    return ym1


def rkl2_hybrid_advance(apply_M, u0, dt, dt_exp, euler_frac, n_euler, n_sub):
    """PAPER.md:341 (Sec. 6): "sub-cycling explicit Euler steps for ~1/4 of the
    time-step and completing the remainder of the step with RKL2", and "sub-cycling
    the RKL2 method within each large time-step":
      n_euler explicit Euler steps u <- u + dte M u, dte = euler_frac dt / n_euler,
      then n_sub RKL2 super-steps of dtr = (1 - euler_frac) dt / n_sub, each with
      s = rkl2_num_stages(dtr, dt_exp) (Eq. 5)."""
    u = np.array(u0, dtype=np.float64)
    if n_euler:
        dte = euler_frac * dt / n_euler
        for _ in range(n_euler):
            u = u + dte * apply_M(u)
    dtr = (1.0 - euler_frac) * dt / n_sub
    s = rkl2_num_stages(dtr, dt_exp)
    for _ in range(n_sub):
        u = rkl2_advance(apply_M, u, dtr, s)
    return u, s


# --------------------------------------------------------------------------
# Backward Euler + PCG  (Sec. 2, Eqs. 2-4, Fig. 1, App. A PC1)
# --------------------------------------------------------------------------


def be_system(op: Operator, dt):
    """Symmetric form of PAPER.md:58 Eq. (4): (I - dt M) u^{n+1} = u^n scaled
    by wV, i.e. A = diag(wV) - dt L (SPD), rhs = wV u^n (DESIGN R7)."""
    return sp.csr_matrix(sp.diags(op.WV) - dt * op.L)


def pcg(A, b, x0, rtol, kmax, return_history=False):
    """PAPER.md:70-92 (Fig. 1) with the point-Jacobi preconditioner PC1
    (P_ii = A_ii, z_i = r_i / P_ii).  DESIGN R8: the last
    line uses z_{k+1}; "Check r_r for convergence" means
    r.z <= rtol^2 * (b . P^-1 b)  (preconditioned residual norm relative to
    the preconditioned right-hand side), tested before every iteration.
    Returns (x, iterations[, history of r.z])."""
    x = np.array(x0, dtype=np.float64)
    P = A.diagonal()
    r = b - A @ x
    z = r / P
    p = z.copy()
    rr = float(r @ z)
    thresh = rtol * rtol * float(b @ (b / P))
    hist = [rr]
    if rr <= thresh:
        return (x, 0, hist) if return_history else (x, 0)
    k = 0
    for k in range(1, kmax + 1):
        y = A @ p
        alpha = rr / float(p @ y)
        x = x + alpha * p
        r = r - alpha * y
        z = r / P
        rold = rr
        rr = float(r @ z)
        hist.append(rr)
        if rr <= thresh:
            break
        beta = rr / rold
        p = beta * p + z
    return (x, k, hist) if return_history else (x, k)


def be_pcg_solve(op: Operator, u_n, dt, rtol=1e-12, kmax=100000):
    """One backward-Euler step of du/dt = M u solved by Jacobi-PCG, x0 = u^n
    (PAPER.md:71).  u_n: grid.shape or (ncomp,)+grid.shape (independent solves).
    Returns (u^{n+1}, iterations per component)."""
    u_n = np.asarray(u_n, dtype=np.float64)
    if u_n.ndim == 4:
        res = [be_pcg_solve(op, x, dt, rtol, kmax) for x in u_n]
        return np.stack([r[0] for r in res]), [r[1][0] for r in res]
    A = be_system(op, dt)
    x, k = pcg(A, op.WV * u_n.ravel(), u_n.ravel(), rtol, kmax)
    return x.reshape(op.grid.shape), [k]
