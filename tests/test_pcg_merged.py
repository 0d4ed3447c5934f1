"""The merged (one-pass, one-reduction) PCG iteration of the CUDA path against
PAPER.md Fig. 1 as the oracle writes it.

The library's default BE solve (DESIGN.md §5.3 "merged PCG", pcg.cuh PH_M)
reorganises Fig. 1 so that an iteration is ONE stencil pass and ONE global
reduction: the pass forms z_k = z_{k-1} - alpha_{k-1} w_{k-1} (w = d y, d = 1/A_ii)
and p_k = z_k + beta_k p_{k-1} on the fly, applies A, and reduces r_k.z_k
(= z_k^2 / d), p_k.y_k, z_k.y_k and w_k.y_k together; the next r.z comes from

    r_{k+1}.z_{k+1} = (r_k - a y_k).d(r_k - a y_k) = r_k.z_k - 2a z_k.y_k + a^2 w_k.y_k.

Round 2 stores no z -- the pass forms p_k from the staged p_{k-2},
w_{k-1}, p_{k-1} -- and updates x every other pass; merged2_pcg / _merged2_exact below
restate that version and pin it the same way.

These host-side tests (no GPU) restate that iteration in numpy / exact rationals,
independently of the CUDA code, and pin it to the oracle's Fig. 1:
  * exact rational arithmetic: identical iterates, alphas, betas and residual
    norms to Fig. 1 on small SPD systems (the reorganisation is an identity);
  * FP64 on the configs' operators: same iteration count (+-1), iterate within the
    residual-stopped uniqueness bound, and the recurrence's r.z within a few ulps
    of r_k.z_k of the true r_{k+1} at every iteration (no drift: the recurrence
    restarts from the pass's own r_k.z_k).
"""
from fractions import Fraction

import numpy as np
import pytest
import scipy.sparse.linalg as spl

import workloads as W
from oracle import core as O


def merged_pcg(A, b, x0, rtol, kmax, hist=None):
    """The CUDA path's merged iteration (capi.cu iteration_m, stencil_tma*.cu
    EPI_PCG_M, pcg.cuh PH_M), in the kernel's order of operations."""
    P = A.diagonal()
    d = 1.0 / P
    x = np.array(x0, dtype=np.float64)
    r0 = b - A @ x
    z = r0 * d                                    # R0 pass: z_0 = r_0 d
    thresh = rtol * rtol * float(b @ (b * d))
    if float(r0 @ z) <= thresh:
        return x, 0
    w = p = None
    alpha = beta = 0.0
    k = 0
    while k < kmax:
        k += 1
        if k > 1:
            z = z - alpha * w                     # z_k = z_{k-1} - alpha_{k-1} d y_{k-1}
            x = x + alpha * p                     # deferred x_k = x_{k-1} + alpha_{k-1} p_{k-1}
            p = z + beta * p
        else:
            p = z.copy()
        y = A @ p
        w = d * y
        rz = float(np.sum(z * z / d))
        pAp, zy, wy = float(p @ y), float(z @ y), float(w @ y)
        alpha = rz / pAp
        rz_next = rz - 2.0 * alpha * zy + alpha * alpha * wy
        if hist is not None:
            r_next = (z - alpha * w) / d          # the true r_{k+1} (only for the check)
            hist.append((rz, rz_next, float(r_next @ (r_next * d))))
        if rz_next <= thresh:
            x = x + alpha * p                     # final deferred update (pcg_xfinal)
            break
        beta = rz_next / rz
    return x, k


# ---------------------------------------------------------------- exact arithmetic
def _fig1_exact(A, b, x0, n):
    """Fig. 1 with the Jacobi preconditioner, exact rationals, n iterations."""
    m = len(b)
    P = [A[i][i] for i in range(m)]
    mv = lambda v: [sum(A[i][j] * v[j] for j in range(m)) for i in range(m)]
    dot = lambda a, c: sum(ai * ci for ai, ci in zip(a, c))
    x = list(x0)
    Ax = mv(x)
    r = [b[i] - Ax[i] for i in range(m)]
    z = [r[i] / P[i] for i in range(m)]
    p = list(z)
    rr = dot(r, z)
    out = []
    for _ in range(n):
        y = mv(p)
        a = rr / dot(p, y)
        x = [x[i] + a * p[i] for i in range(m)]
        r = [r[i] - a * y[i] for i in range(m)]
        z = [r[i] / P[i] for i in range(m)]
        rold, rr = rr, dot(r, z)
        if rr == 0:
            out.append((a, None, rr, list(x)))
            break
        beta = rr / rold
        p = [z[i] + beta * p[i] for i in range(m)]
        out.append((a, beta, rr, list(x)))
    return out


def _merged_exact(A, b, x0, n):
    """The merged iteration, exact rationals (same order as merged_pcg)."""
    m = len(b)
    d = [1 / A[i][i] for i in range(m)]
    mv = lambda v: [sum(A[i][j] * v[j] for j in range(m)) for i in range(m)]
    dot = lambda a, c: sum(ai * ci for ai, ci in zip(a, c))
    x = list(x0)
    Ax = mv(x)
    z = [(b[i] - Ax[i]) * d[i] for i in range(m)]
    out = []
    w = p = None
    alpha = beta = Fraction(0)
    for k in range(1, n + 1):
        if k > 1:
            z = [z[i] - alpha * w[i] for i in range(m)]
            x = [x[i] + alpha * p[i] for i in range(m)]
            p = [z[i] + beta * p[i] for i in range(m)]
        else:
            p = list(z)
        y = mv(p)
        w = [d[i] * y[i] for i in range(m)]
        rz = sum(z[i] * z[i] / d[i] for i in range(m))
        alpha = rz / dot(p, y)
        rz_next = rz - 2 * alpha * dot(z, y) + alpha * alpha * dot(w, y)
        xk = [x[i] + alpha * p[i] for i in range(m)]     # x_{k} of Fig. 1's numbering
        if rz_next == 0:
            out.append((alpha, None, rz_next, xk))
            break
        beta = rz_next / rz
        out.append((alpha, beta, rz_next, xk))
    return out


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_merged_iteration_is_fig1_in_exact_arithmetic(seed):
    rng = np.random.default_rng(seed)
    m = 6
    # SPD, diagonally dominant, integer entries: a small stand-in for wV - dt L
    B = rng.integers(-3, 4, size=(m, m))
    S = B @ B.T + np.diag(rng.integers(1, 5, size=m)) + 3 * np.eye(m, dtype=int)
    A = [[Fraction(int(S[i, j])) for j in range(m)] for i in range(m)]
    b = [Fraction(int(v)) for v in rng.integers(-9, 10, size=m)]
    x0 = [Fraction(int(v), 7) for v in rng.integers(-5, 6, size=m)]
    f1 = _fig1_exact(A, b, x0, m)
    mg = _merged_exact(A, b, x0, m)
    assert len(f1) == len(mg)
    for (a1, b1, r1, x1), (a2, b2, r2, x2) in zip(f1, mg):
        assert a1 == a2 and b1 == b2 and r1 == r2 and x1 == x2
    # CG on an m x m SPD system terminates in at most m steps with the exact solution
    Sf = np.array(S, dtype=float)
    assert np.allclose([float(v) for v in mg[-1][3]], np.linalg.solve(Sf, [float(v) for v in b]), rtol=1e-12)


# ---------------------------------------------------------------- FP64 on the configs' operators
def _system(case):
    if case == "c1":
        cfg = W.make_config("c1_spitzer64", shape=(16, 15, 24))
        g = cfg["grid"]
        kap = O.spitzer_face_kappa(g, cfg["T"].numpy(), cfg["kappa0"], cfg["T_cut"])
        op = O.Operator(g, kap, cfg["b"].numpy())
        u, ratio = cfg["T"].numpy(), 100.0
    elif case == "c2":
        cfg = W.make_config("c2_visc64", shape=(16, 15, 24))
        g = cfg["grid"]
        op = O.Operator(g, [f.numpy() for f in cfg["visc_faces"]], None, cfg["rho"].numpy())
        u, ratio = cfg["v"].numpy()[1], 500.0
    else:
        cfg = W.make_config("c0_heat32")
        g = cfg["grid"]
        op = O.Operator(g, [f.numpy() for f in cfg["faces"]])
        u, ratio = cfg["u"].numpy(), 50.0
    dt = ratio * O.dt_euler(op)
    A = O.be_system(op, dt).tocsr()
    return op, A, op.WV * u.ravel(), u.ravel()


@pytest.mark.parametrize("case", ["c0", "c1", "c2"])
def test_merged_iteration_matches_oracle_fp64(case):
    op, A, b, x0 = _system(case)
    ref, k_ref = O.pcg(A, b, x0, 1e-12, 100000)
    hist = []
    x, k = merged_pcg(A, b, x0, 1e-12, 100000, hist)
    assert abs(k - k_ref) <= 1, (k, k_ref)
    exact = spl.spsolve(A.tocsc(), b)
    tol = max(1e-11, np.linalg.norm(ref - exact) / np.linalg.norm(exact))
    assert np.linalg.norm(x - ref) <= 2 * tol * np.linalg.norm(ref)
    # the recurrence's r.z agrees with the true r_{k+1}.z_{k+1} to rounding of r_k.z_k
    # (it restarts from each pass's own sum: no drift over the ~100 iterations)
    for rz, est, true in hist:
        assert abs(est - true) <= 1e-12 * rz, (rz, est, true)


# ---------------------------------------------------------------- round 2: no z stored, x in pairs
def merged2_pcg(A, b, x0, rtol, kmax, modes=None, hist=None):
    """The CUDA path's merged iteration as of round 2 (DESIGN.md §5.3 "No z stored",
    "x in pairs"; pcg.cuh PH_M, stencil_tma*.cu EPI_PCG_M, aux.cu pcg_xfinal_kernel), in
    the kernels' order of operations: the pass stages p_{k-2}, w_{k-1}, p_{k-1} and forms
      z_k = (p_{k-1} - beta_{k-1} p_{k-2}) - alpha_{k-1} w_{k-1},  p_k = z_k + beta_k p_{k-1};
    x is updated every other pass (a skipped pass, then a catch-up
    x_k = x_{k-2} + alpha_{k-1} p_{k-1} + alpha_{k-2} p_{k-2}); the final pass adds what x
    still owes.  `modes` collects each pass's x mode (0 normal, 1 skip, 2 catch-up)."""
    P = A.diagonal()
    d = 1.0 / P
    x = np.array(x0, dtype=np.float64)
    z0 = (b - A @ x) * d
    thresh = rtol * rtol * float(b @ (b * d))
    if float(np.sum(z0 * z0 / d)) <= thresh:
        return x, 0
    pk = {0: z0}                                  # p_0 := z_0 (coefficient beta_1 = 0 at k = 2)
    w = None
    ax = beta = bprev = 0.0
    xm, cxp, cxz = 0, 0.0, 0.0
    k = iters = 0
    while k < kmax:
        k += 1
        if k == 1:
            z = z0
            p = z0.copy()
        else:
            f0, f1, f2 = pk[k - 2], w, pk[k - 1]
            z = (f2 - bprev * f0) - ax * f1
            p = z + beta * f2
            if xm == 0:
                x = x + ax * f2
            elif xm == 2:
                x = (x + cxp * f2) + cxz * f0
        if modes is not None:
            modes.append(xm if k > 1 else 0)
        pk[k] = p
        y = A @ p
        w = d * y
        rz = float(np.sum(z * z / d))
        pAp, zy, wy = float(p @ y), float(z @ y), float(w @ y)
        mk = xm
        if rz <= thresh:                          # (the pass's own r.z meets the test)
            if mk == 1:
                x = x + ax * pk[k - 1]
            return x, iters
        a_prev = ax
        bprev = beta
        alpha = rz / pAp
        rz_next = rz - 2.0 * alpha * zy + alpha * alpha * wy
        iters = k
        ax = alpha
        if hist is not None:
            hist.append((alpha, rz_next))
        if rz_next <= thresh:
            if mk == 1:
                x = x + a_prev * pk[k - 1]
            return x + alpha * p, iters
        beta = rz_next / rz
        if mk == 1:
            xm, cxp, cxz = 2, alpha, a_prev
        else:
            xm = 1
        pk.pop(k - 3, None)
    return x, iters


def _merged2_exact(A, b, x0, n):
    """merged2_pcg in exact rationals for n passes; per pass (alpha, beta, r.z next) and
    the x the final pass would return after it."""
    m = len(b)
    d = [1 / A[i][i] for i in range(m)]
    mv = lambda v: [sum(A[i][j] * v[j] for j in range(m)) for i in range(m)]
    dot = lambda a, c: sum(ai * ci for ai, ci in zip(a, c))
    x = list(x0)
    Ax = mv(x)
    z0 = [(b[i] - Ax[i]) * d[i] for i in range(m)]
    pk = {0: z0}
    w = None
    ax = beta = bprev = Fraction(0)
    xm, cxp, cxz = 0, Fraction(0), Fraction(0)
    out = []
    for k in range(1, n + 1):
        if k == 1:
            z, p = z0, list(z0)
        else:
            f0, f1, f2 = pk[k - 2], w, pk[k - 1]
            z = [(f2[i] - bprev * f0[i]) - ax * f1[i] for i in range(m)]
            p = [z[i] + beta * f2[i] for i in range(m)]
            if xm == 0:
                x = [x[i] + ax * f2[i] for i in range(m)]
            elif xm == 2:
                x = [(x[i] + cxp * f2[i]) + cxz * f0[i] for i in range(m)]
        pk[k] = p
        y = mv(p)
        w = [d[i] * y[i] for i in range(m)]
        rz = sum(z[i] * z[i] / d[i] for i in range(m))
        a_prev, bprev = ax, beta
        alpha = rz / dot(p, y)
        rz_next = rz - 2 * alpha * dot(z, y) + alpha * alpha * dot(w, y)
        ax = alpha
        # the final pass after this one: x += [alpha_{k-1} p_{k-1}] + alpha_k p_k
        xf = list(x)
        if xm == 1:
            xf = [xf[i] + a_prev * pk[k - 1][i] for i in range(m)]
        xf = [xf[i] + alpha * p[i] for i in range(m)]
        if rz_next == 0:
            out.append((alpha, None, rz_next, xf))
            break
        beta = rz_next / rz
        out.append((alpha, beta, rz_next, xf))
        xm, cxp, cxz = (2, alpha, a_prev) if xm == 1 else (1, cxp, cxz)
    return out


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_round2_iteration_is_fig1_in_exact_arithmetic(seed):
    """No z stored + x in pairs: identical alphas, betas, residual norms and iterates to
    Fig. 1 in exact arithmetic, for every pass (skipped or catch-up)."""
    rng = np.random.default_rng(seed)
    m = 7
    B = rng.integers(-3, 4, size=(m, m))
    S = B @ B.T + np.diag(rng.integers(1, 5, size=m)) + 3 * np.eye(m, dtype=int)
    A = [[Fraction(int(S[i, j])) for j in range(m)] for i in range(m)]
    b = [Fraction(int(v)) for v in rng.integers(-9, 10, size=m)]
    x0 = [Fraction(int(v), 7) for v in rng.integers(-5, 6, size=m)]
    f1 = _fig1_exact(A, b, x0, m)
    mg = _merged2_exact(A, b, x0, m)
    assert len(f1) == len(mg)
    for (a1, b1, r1, x1), (a2, b2, r2, x2) in zip(f1, mg):
        assert a1 == a2 and b1 == b2 and r1 == r2 and x1 == x2


@pytest.mark.parametrize("case", ["c0", "c1", "c2"])
def test_round2_iteration_matches_oracle_fp64(case):
    """FP64 on the configs' operators: iteration count +-1 and the iterate within the
    residual-stopped uniqueness bound of the oracle's Fig. 1 at rtol 1e-12; at rtol 1e-15
    within 1e-11 of the direct solve (the GPU tests' fixed bar, DESIGN R12); the x modes
    alternate skip / catch-up after the first two passes."""
    op, A, b, x0 = _system(case)
    ref, k_ref = O.pcg(A, b, x0, 1e-12, 100000)
    modes = []
    x, k = merged2_pcg(A, b, x0, 1e-12, 100000, modes)
    assert abs(k - k_ref) <= 1, (k, k_ref)
    exact = spl.spsolve(A.tocsc(), b)
    tol = max(1e-11, np.linalg.norm(ref - exact) / np.linalg.norm(exact))
    assert np.linalg.norm(x - ref) <= 2 * tol * np.linalg.norm(ref)
    assert modes[:3] == [0, 1, 2] and all(modes[i] == (1 if i % 2 else 2) for i in range(1, len(modes)))
    x15, _ = merged2_pcg(A, b, x0, 1e-15, 100000)
    assert np.linalg.norm(x15 - exact) <= 1e-11 * np.linalg.norm(exact)
