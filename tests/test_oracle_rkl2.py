"""Pins for the oracle's RKL2 stage count, coefficients and recursion.

Independent of the oracle's own formulas: brute-force stability inequality,
the Legendre closed form of the RKL2 stability polynomial (numpy's Legendre
routine), order conditions, and values printed in PAPER.md (tests/golden).
"""
import json
import math
import os

import numpy as np
import pytest
from numpy.polynomial import legendre

from oracle import core as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_claims.json")))


def _legendre_R(s, z):
    """RKL2 stability polynomial in closed form (Meyer, Balsara & Aslam 2014,
    the RKL2 reference cited at PAPER.md:31): R_s(z) = 1 - b_s + b_s P_s(1 + w1 z),
    b_s = (s^2+s-2)/(2 s (s+1)), w1 = 4/(s^2+s-2).  Written from that paper, not
    from oracle.rkl2_coeffs."""
    bs = (s * s + s - 2.0) / (2.0 * s * (s + 1.0))
    w1 = 4.0 / (s * s + s - 2.0)
    return 1.0 - bs + bs * legendre.legval(1.0 + w1 * np.asarray(z), [0] * s + [1])


def _scalar_G(s, z):
    z = np.asarray(z, dtype=np.float64)
    return O.rkl2_advance(lambda u: z * u, np.ones_like(z), 1.0, s)


def test_stage_count_brute_force():
    # PAPER.md:142 Eq.(5): smallest s >= 2 with (s^2+s-2)/4 >= dt/dt_exp
    for ratio in np.logspace(-1, 4, 400):
        s = O.rkl2_num_stages(ratio, 1.0)
        smin = next(t for t in range(2, 1000) if (t * t + t - 2) / 4.0 >= ratio * (1 - 1e-15))
        assert s == smin, (ratio, s, smin)


def test_stage_count_spot_values():
    assert O.rkl2_num_stages(1.0, 1.0) == 2
    assert O.rkl2_num_stages(10.0, 1.0) == 6      # exactly at the stability boundary
    assert O.rkl2_num_stages(100.0, 1.0) == 20
    assert O.rkl2_num_stages(300.0, 1.0) == 35
    assert O.rkl2_num_stages(500.0, 1.0) == 45
    assert O.rkl2_num_stages(1e-9, 1.0) == 2      # floor of the scheme
    assert O.rkl2_num_stages(100.0, 1.0, force_odd=True) == 21


def test_stage_scaling_sqrt():
    # s ~ 1/dx while dt/dt_E ~ 1/dx^2 -> s(4r)/s(r) -> 2
    r = 1e6
    assert abs(O.rkl2_num_stages(4 * r, 1.0) / O.rkl2_num_stages(r, 1.0) - 2.0) < 1e-3


@pytest.mark.parametrize("s", [2, 3, 4, 5, 10, 20, 35, 45, 63])
def test_recursion_matches_legendre_closed_form(s):
    zmin = -(s * s + s - 2) / 2.0
    z = np.linspace(zmin, 0.0, 257)
    G = _scalar_G(s, z)
    R = _legendre_R(s, z)
    assert np.max(np.abs(G - R)) < 1e-12 * max(1.0, s)


def test_gamma_reading_is_the_b_jm1_one():
    """DESIGN R6: Fig. 2 prints (b_k - 1) mu~_k; only (b_{k-1} - 1) mu~_k reproduces
    the closed form / second order.  Demonstrate the printed index fails."""
    s = 10
    c = O.rkl2_coeffs(s)
    z = np.linspace(-(s * s + s - 2) / 2.0, 0.0, 65)
    y0 = np.ones_like(z)
    ym2, ym1 = y0, y0 + c["mut"][1] * z * y0
    for j in range(2, s + 1):
        g_alt = (c["b"][j] - 1.0) * c["mut"][j]
        yj = c["mu"][j] * ym1 + c["nu"][j] * ym2 + (1 - c["mu"][j] - c["nu"][j]) * y0 \
            + c["mut"][j] * z * ym1 + g_alt * z * y0
        ym2, ym1 = ym1, yj
    assert np.max(np.abs(ym1 - _legendre_R(s, z))) > 1e-3


@pytest.mark.parametrize("s", [2, 5, 20, 45])
def test_order_conditions(s):
    # G(0)=1, G'(0)=1, G''(0)=1 (second order), by finite differences
    h = 1e-3
    g = _scalar_G(s, np.array([-2 * h, -h, 0.0, h, 2 * h]))
    assert abs(g[2] - 1.0) < 1e-14
    d1 = (g[3] - g[1]) / (2 * h)
    d2 = (g[3] - 2 * g[2] + g[1]) / h ** 2
    assert abs(d1 - 1.0) < 1e-6 and abs(d2 - 1.0) < 1e-4


@pytest.mark.parametrize("s", [2, 3, 7, 20, 35, 63])
def test_stability_interval(s):
    # |G(z)| <= 1 on z in [-(s^2+s-2)/2, 0]  (dt <= dt_E (s^2+s-2)/4, dt_E = 2/|lam|)
    z = np.linspace(-(s * s + s - 2) / 2.0, 0.0, 4001)
    assert np.max(np.abs(_scalar_G(s, z))) <= 1.0 + 1e-12


def test_identity_when_M_zero():
    u = np.random.default_rng(0).normal(size=50)
    out = O.rkl2_advance(lambda x: 0.0 * x, u, 3.7, 17)
    assert np.max(np.abs(out - u)) < 1e-14 * np.max(np.abs(u))


def test_paper_high_mode_damping_claim():
    g = GOLD["rkl2_high_mode_damping"]
    ratio = g["ratio"]
    z = -2.0 * ratio * math.sin(g["k_dx"] / 2) ** 2  # 1-D mode: z = -2 r sin^2(k dx / 2)
    s = O.rkl2_num_stages(ratio, 1.0)
    G = abs(_scalar_G(s, np.array([z]))[0])
    lo, hi = g["accept_interval"]
    assert lo <= G <= hi, G
    # BE for comparison: 1/(1 - z) = 1/1001
    assert abs(1.0 / (1.0 - z) - 1.0 / 1001.0) < 1e-15


def test_paper_not_l_stable_and_low_mode_accuracy():
    for ratio in GOLD["rkl2_not_l_stable"]["ratios"]:
        s = O.rkl2_num_stages(ratio, 1.0)
        z = -2.0 * ratio
        assert abs(_scalar_G(s, np.array([z]))[0]) > 0.25
        assert abs(1.0 / (1.0 - z)) < 0.1
    g = GOLD["rkl2_low_mode_accuracy"]
    s = O.rkl2_num_stages(g["ratio"], 1.0)
    kdx = np.linspace(1e-3, g["k_dx_max"], 50)
    z = -2.0 * g["ratio"] * np.sin(kdx / 2) ** 2
    err_rkl2 = np.abs(_scalar_G(s, z) - np.exp(z))
    err_be = np.abs(1.0 / (1.0 - z) - np.exp(z))
    assert np.all(err_rkl2 < err_be)


def test_second_order_in_time():
    """Temporal order on a stiff diagonal system: error vs exp(dt*lam) quarters
    when dt halves (two steps)."""
    lam = -np.logspace(-1, 2, 40)
    dt_exp = 2.0 / np.max(np.abs(lam))
    T = 0.05
    errs = []
    for nsteps in (4, 8, 16):
        dt = T / nsteps
        s = O.rkl2_num_stages(dt, dt_exp)
        u = np.ones_like(lam)
        for _ in range(nsteps):
            u = O.rkl2_advance(lambda x: lam * x, u, dt, s)
        errs.append(np.linalg.norm(u - np.exp(lam * T)))
    order = math.log2(errs[1] / errs[2])
    assert 1.7 < order < 2.6, errs


# ---------------------------------------------------------------- PAPER.md:341 remedies
def _hybrid_G(z_over_dtexp, ratio, euler_frac, n_euler, n_sub):
    """Amplification of the oracle's hybrid on the scalar ODE u' = lam u, with
    lam = z_over_dtexp / dt_exp (dt_exp = 1)."""
    lam = np.asarray(z_over_dtexp, dtype=np.float64)
    u, s = O.rkl2_hybrid_advance(lambda u: lam * u, np.ones_like(lam), ratio, 1.0, euler_frac, n_euler, n_sub)
    return u, s


@pytest.mark.parametrize("ratio,frac,n_euler,n_sub", [(500.0, 0.25, 250, 1), (50.0, 0.25, 25, 2), (300.0, 0.0, 0, 10),
                                                       (100.0, 0.5, 100, 3)])
def test_hybrid_closed_form(ratio, frac, n_euler, n_sub):
    """The hybrid applied to u' = lam u is (1 + dte lam)^n_euler R_s(dtr lam)^n_sub with
    R_s the Legendre closed form -- written from the definition, not the oracle."""
    z = -np.linspace(0.0, 2.0, 41)                           # lam dt_exp over the stable range
    got, s = _hybrid_G(z, ratio, frac, n_euler, n_sub)
    dte = frac * ratio / n_euler if n_euler else 0.0
    dtr = (1 - frac) * ratio / n_sub
    smin = next(t for t in range(2, 100000) if (t * t + t - 2) / 4.0 >= dtr * (1 - 1e-15))
    assert s == smin
    want = (1.0 + dte * z) ** n_euler * _legendre_R(s, dtr * z) ** n_sub
    np.testing.assert_allclose(got, want, rtol=1e-10, atol=1e-13)


def test_hybrid_reduces_to_rkl2():
    z = -np.linspace(0.0, 2.0, 17)
    got, s = _hybrid_G(z, 123.0, 0.0, 0, 1)
    assert s == O.rkl2_num_stages(123.0, 1.0)
    np.testing.assert_allclose(got, _scalar_G(s, 123.0 * z), rtol=1e-13, atol=1e-15)


def test_paper_euler_prefix_damps_high_modes_more_than_be():
    """explicit Euler over ~1/4 of the step 'damps high modes more than
    even a full step with BE' (Fig. 8 ratio 500, dte = dt_exp/2): over the upper half
    of the discrete spectrum the hybrid's amplification is below BE's 1/(1 - dt lam)."""
    ratio = GOLD["rkl2_high_mode_damping"]["ratio"]
    z = -np.linspace(1.0, 2.0, 101)                          # lam dt_exp, upper half
    got, _ = _hybrid_G(z, ratio, 0.25, int(0.25 * ratio / 0.5), 1)
    be = 1.0 / (1.0 - ratio * z)
    assert np.all(np.abs(got) <= np.abs(be))
    # ... while plain RKL2 at that ratio leaves ~0.5 there
    s = O.rkl2_num_stages(ratio, 1.0)
    assert np.abs(_scalar_G(s, ratio * z[-1])) > 0.3


def test_paper_rkl2_subcycling_approaches_be():
    """sub-cycling RKL2 (~10 sub-cycles) gives a solution close to BE:
    the high-mode amplification moves from ~0.5 (one super-step) to near BE's."""
    ratio = 500.0
    z = -np.linspace(1.5, 2.0, 51)
    one = np.abs(_scalar_G(O.rkl2_num_stages(ratio, 1.0), ratio * z))
    sub, _ = _hybrid_G(z, ratio, 0.0, 0, 10)
    be = np.abs(1.0 / (1.0 - ratio * z))
    assert np.max(np.abs(np.abs(sub) - be)) < 0.25 * np.min(np.abs(one - be))
