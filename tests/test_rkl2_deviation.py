"""The deviation form of the RKL2 stages used by the CUDA path (DESIGN.md §5.3,
`sts_grid_set_rkl2_deviation`) against PAPER.md Fig. 2 as the oracle writes it.

With M linear over the super-step, Y_j = Y0 + D_j turns Fig. 2's stage into

    D_j = mu_j D_{j-1} + nu_j D_{j-2} + mu~_j dt M D_{j-1} + (mu~_j + gamma~_j) dt M Y0,

D_0 = 0, D_1 = mu~_1 dt M Y0, and the last stage returns Y0 + D_s with Fig. 2's own
arithmetic.  These host-side tests restate that recurrence (independently of the
CUDA code) and pin it to the oracle: identical stages in exact rational arithmetic,
and FP64 agreement to rounding on configs[0] and a 3-component viscosity operator.
"""
from fractions import Fraction

import numpy as np
import pytest

import workloads as W
from oracle import core as O


def deviation_rkl2(apply_M, u0, dt, s):
    """The CUDA path's stage sequence (capi.cu rkl2_core with deviation form)."""
    c = O.rkl2_coeffs(s)
    y0 = np.array(u0, dtype=np.float64)
    M0 = apply_M(y0)
    dm1 = c["mut"][1] * dt * M0            # D_1 (the first-stage kernel with a0 = 0)
    dm2 = None                             # D_0 = 0
    for j in range(2, s):
        nu = c["nu"][j] if dm2 is not None else 0.0
        d = (c["mu"][j] * dm1 + nu * (dm2 if dm2 is not None else dm1) + c["mut"][j] * dt * apply_M(dm1)
             + (c["mut"][j] + c["gt"][j]) * dt * M0)
        dm2, dm1 = dm1, d
    # the last stage: the printed stage's operands with Y0 added back (c2 = 1)
    j = s
    nu = c["nu"][j] if dm2 is not None else 0.0
    return (c["mu"][j] * dm1 + nu * (dm2 if dm2 is not None else dm1) + 1.0 * y0 + c["mut"][j] * dt * apply_M(dm1)
            + (c["mut"][j] + c["gt"][j]) * dt * M0)


def _fig2_exact(A, u0, dt, s):
    # the oracle's FP64 coefficients, taken exactly (Fraction of a double is exact)
    c = {k: [Fraction(float(v)) for v in O.rkl2_coeffs(s)[k]] for k in ("mu", "nu", "mut", "gt")}
    mv = lambda v: [sum(A[i][k] * v[k] for k in range(len(v))) for i in range(len(v))]  # noqa: E731
    y0 = list(u0)
    M0 = mv(y0)
    ym2, ym1 = y0, [y0[i] + c["mut"][1] * dt * M0[i] for i in range(len(y0))]
    out = [ym1]
    for j in range(2, s + 1):
        My = mv(ym1)
        yj = [c["mu"][j] * ym1[i] + c["nu"][j] * ym2[i] + (1 - c["mu"][j] - c["nu"][j]) * y0[i]
              + c["mut"][j] * dt * My[i] + c["gt"][j] * dt * M0[i] for i in range(len(y0))]
        ym2, ym1 = ym1, yj
        out.append(yj)
    return out


def _dev_exact(A, u0, dt, s):
    # the oracle's FP64 coefficients, taken exactly (Fraction of a double is exact)
    c = {k: [Fraction(float(v)) for v in O.rkl2_coeffs(s)[k]] for k in ("mu", "nu", "mut", "gt")}
    n = len(u0)
    mv = lambda v: [sum(A[i][k] * v[k] for k in range(n)) for i in range(n)]  # noqa: E731
    M0 = mv(list(u0))
    d = [[Fraction(0)] * n, [c["mut"][1] * dt * M0[i] for i in range(n)]]
    for j in range(2, s + 1):
        Md = mv(d[j - 1])
        d.append([c["mu"][j] * d[j - 1][i] + c["nu"][j] * d[j - 2][i] + c["mut"][j] * dt * Md[i]
                  + (c["mut"][j] + c["gt"][j]) * dt * M0[i] for i in range(n)])
    return [[u0[i] + dj[i] for i in range(n)] for dj in d[1:]]


@pytest.mark.parametrize("s", [2, 3, 7])
def test_deviation_form_is_fig2_in_exact_arithmetic(s):
    rng = np.random.default_rng(s)
    n = 5
    B = rng.integers(-3, 4, size=(n, n))
    A = [[Fraction(int(v)) for v in row] for row in -(B @ B.T) - np.eye(n, dtype=int)]   # M <= 0
    u0 = [Fraction(int(v), 3) for v in rng.integers(-6, 7, size=n)]
    dt = Fraction(1, 40)
    assert _fig2_exact(A, u0, dt, s) == _dev_exact(A, u0, dt, s)   # every stage Y_j = Y0 + D_j


@pytest.mark.parametrize("case", ["c0", "visc3"])
def test_deviation_form_matches_oracle_fp64(case):
    if case == "c0":
        cfg = W.make_config("c0_heat32")
        op = O.Operator(cfg["grid"], [f.numpy() for f in cfg["faces"]])
        u0, ratio = cfg["u"].numpy(), 50.0
        apply_M = lambda x: (op.M @ x.ravel()).reshape(x.shape)  # noqa: E731
    else:
        cfg = W.make_config("c2_visc64", shape=(12, 11, 16))
        op = O.Operator(cfg["grid"], [f.numpy() for f in cfg["visc_faces"]], None, cfg["rho"].numpy())
        u0, ratio = cfg["v"].numpy(), 500.0
        apply_M = op.apply
    dte = O.dt_euler(op)
    dt = ratio * dte
    s = O.rkl2_num_stages(dt, dte)
    ref = O.rkl2_advance(apply_M, u0, dt, s)
    got = deviation_rkl2(apply_M, u0, dt, s)
    assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)
