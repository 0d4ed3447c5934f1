"""GPU parity at BASELINE.json's FULL sizes, in bench.py's launch configuration
(one Grid over the whole grid, TMA kernels on, device-resident inputs).

The oracle cannot hold a 268M-cell operator, so (task ③ / DESIGN.md §0):
  * RKL2 and F(u): sampled outputs.  After s stages a cell depends only on the
    cells within s of it (27-point stencil, radius 1 per stage), so the oracle
    runs the same super-step (same dt, same s) on the index box of half-width
    s + 2 around each sampled cell -- with the TRUE domain walls where the box
    touches them and periodic wrap in phi -- and its centre value must match.
  * BE + PCG (a global solve): the GPU iterate must satisfy the ORACLE's linear
    system on EVERY row -- r = b - A x from the plain-C oracle's matrix-free row
    gather (OpenMP), in the preconditioned norm of the stopping test (DESIGN R8).
Samples include the r_min wall, the theta poles, the periodic phi seam, the steep
transition-region ramp and the interior.
"""
import os

import numpy as np
import pytest
import torch

import workloads as W
from oracle import core as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import __graft_entry__ as e
    e.build()
    return torch.device("cuda", 0)


def _gather(t, idx):
    """t[..., I, J, K] for the index arrays of W.subgrid (on the device), to numpy."""
    I, J, K = (torch.as_tensor(a, device=t.device) for a in idx)
    x = t.index_select(-3, I).index_select(-2, J).index_select(-1, K)
    return x.cpu().numpy()


SAMPLES = [(0, 0, 0), (2, 255, 1023), (6, 511, 512), (300, 130, 77), (511, 300, 1000)]


@pytest.fixture(scope="module")
def c4(dev):
    from paper_1610_01265_b200 import sts
    cfg = W.make_config("c4_scale512", device=dev)
    G = sts.Grid.from_grid(cfg["grid"])
    return cfg, G


def test_c4_conduction_rkl2_sampled(dev, c4):
    from paper_1610_01265_b200 import sts
    cfg, G = c4
    g = cfg["grid"]
    T, b = cfg["T"], cfg["b"]
    k = G.face_kappa_spitzer(T, cfg["kappa0"], cfg["T_cut"])
    dte = G.dt_euler("aniso", k, b)
    dt = 300.0 * dte
    s = sts.rkl2_num_stages(dt, dte)
    assert s == O.rkl2_num_stages(dt, dte)
    out = G.rkl2_advance("aniso", T, k, b, None, dt, s)
    F = G.op_apply("aniso", T, k, b)
    torch.cuda.synchronize()
    for c in SAMPLES:
        sub, idx, loc = W.subgrid(g, c, s + 2)
        Ts, bs = _gather(T, idx), _gather(b, idx)
        kap = O.spitzer_face_kappa(sub, Ts, cfg["kappa0"], cfg["T_cut"])
        op = O.Operator(sub, kap, bs)
        # Gershgorin bound holds at every row of the box (dt_exp is the global minimum)
        rows = np.asarray(abs(op.M).sum(axis=1)).ravel()
        assert rows.max() <= (2.0 / dte) * (1 + 1e-12)
        ref = O.rkl2_advance(lambda x: (op.M @ x.ravel()).reshape(x.shape), Ts, dt, s)[loc]
        got = float(out[c].item())
        assert abs(got - ref) <= 1e-11 * abs(ref), (c, got, ref)
        fref = op.apply(Ts)[loc]
        scale = np.abs(op.apply(Ts)).max()
        assert abs(float(F[c].item()) - fref) <= 1e-12 * scale, (c, float(F[c].item()), fref)


def test_c4_viscosity_rkl2_sampled(dev, c4):
    from paper_1610_01265_b200 import sts
    cfg, G = c4
    g = cfg["grid"]
    kv, rho, v = cfg["visc_faces"], cfg["rho"], cfg["v"]
    dte = G.dt_euler("iso", kv, None, rho)
    dt = 300.0 * dte
    s = sts.rkl2_num_stages(dt, dte)
    out = G.rkl2_advance("iso", v, kv, None, rho, dt, s)
    torch.cuda.synchronize()
    for c in SAMPLES[:3]:
        sub, idx, loc = W.subgrid(g, c, s + 2)
        ks = [_gather(x, idx) for x in kv]
        # faces leaving the box carry no flux in the oracle; they lie outside the
        # domain of dependence of the centre cell
        op = O.Operator(sub, ks, None, _gather(rho, idx))
        ref = O.rkl2_advance(op.apply, _gather(v, idx), dt, s)
        for q in range(3):
            got = float(out[(q,) + tuple(c)].item())
            r = ref[(q,) + tuple(loc)]
            assert abs(got - r) <= 1e-11 * max(abs(r), np.abs(ref[q]).max() * 1e-3), (c, q, got, r)


def _full_check(g, un, x, kap, b, w, dt, rtol, dte=None):
    """The GPU iterate x against the ORACLE's backward-Euler system over the WHOLE grid
    (oracle/c oc_check_full: every row of L gathered matrix-free from its vertices /
    faces, OpenMP): the stopping test of DESIGN R8 in the preconditioned norm, with a
    factor 2 for the recurrence-vs-true residual gap, ||r||_{P^-1} <= 2 rtol ||b||_{P^-1},
    per component; and, if dte is given, the oracle's full-grid Gershgorin dt_exp
     against the GPU's."""
    from oracle import c_oracle as C
    C.set_threads(os.cpu_count() or 1)
    res, lam = C.check_full(g, un, kap, b, w, x, dt)
    for q, (num, den, mx) in enumerate(res):
        assert num <= (2.0 * rtol) ** 2 * den, (q, num, den, (num / den) ** 0.5)
    if dte is not None:
        assert abs(2.0 / lam - dte) <= 1e-12 * dte, (2.0 / lam, dte)
    return [((num / den) ** 0.5, mx) for num, den, mx in res]


def test_c4_pcg_full_grid_residual(dev, c4):
    """configs[4] at full size, bench.py's launch configuration: conduction and viscosity
    BE + Jacobi-PCG iterates checked against the oracle system on all 268M rows."""
    from oracle import c_oracle as C
    cfg, G = c4
    g = cfg["grid"]
    T, b = cfg["T"], cfg["b"]
    k = G.face_kappa_spitzer(T, cfg["kappa0"], cfg["T_cut"])
    dte = G.dt_euler("aniso", k, b)
    dt = 300.0 * dte
    x, it = G.be_pcg_solve("aniso", T, k, b, None, dt, 1e-12, 50000)
    assert 0 < it[0] < 50000
    del k
    Th, bh, xh = T.cpu().numpy(), b.cpu().numpy(), x.cpu().numpy()
    del x
    torch.cuda.empty_cache()
    C.set_threads(os.cpu_count() or 1)
    kap = C.face_kappa(g, Th, cfg["kappa0"], cfg["T_cut"])
    print("c4 conduction: iterations", it, "(||r||/||b||_P, max|r|/max|b|) =",
          _full_check(g, Th, xh, kap, bh, None, dt, 1e-12, dte))
    del Th, bh, xh, kap
    kv, rho, v = cfg["visc_faces"], cfg["rho"], cfg["v"]
    dtev = G.dt_euler("iso", kv, None, rho)
    xv, itv = G.be_pcg_solve("iso", v, kv, None, rho, 300.0 * dtev, 1e-12, 50000)
    assert all(0 < i < 50000 for i in itv)
    print("c4 viscosity: iterations", itv, _full_check(g, v.cpu().numpy(), xv.cpu().numpy(),
                                                        [f.cpu().numpy() for f in kv], None, rho.cpu().numpy(),
                                                        300.0 * dtev, 1e-12, dtev))


def test_c3_dt_sweep_stages_and_iterations(dev):
    """BASELINE configs[3]: 256 x 256 x 512, dt/dt_exp in {10, 100, 1000}: stage
    counts follow Eq. (5) exactly, PCG iteration counts grow with dt, every BE iterate
    passes the oracle system's stopping test on the whole grid, the oracle's full-grid
    Gershgorin dt_exp equals the GPU's, and the sampled RKL2 result matches the oracle
    at the smallest ratio."""
    from paper_1610_01265_b200 import sts
    from oracle import c_oracle as C
    cfg = W.make_config("c3_spitzer256", device=dev)
    g = cfg["grid"]
    G = sts.Grid.from_grid(g)
    T, b = cfg["T"], cfg["b"]
    k = G.face_kappa_spitzer(T, cfg["kappa0"], cfg["T_cut"])
    dte = G.dt_euler("aniso", k, b)
    Th, bh = T.cpu().numpy(), b.cpu().numpy()
    C.set_threads(os.cpu_count() or 1)
    kap = C.face_kappa(g, Th, cfg["kappa0"], cfg["T_cut"])
    rec = {}
    for ratio in (10.0, 100.0, 1000.0):
        dt = ratio * dte
        s = sts.rkl2_num_stages(dt, dte)
        assert s == O.rkl2_num_stages(dt, dte)
        x, it = G.be_pcg_solve("aniso", T, k, b, None, dt, 1e-12, 50000)
        rec[ratio] = (s, it[0], _full_check(g, Th, x.cpu().numpy(), kap, bh, None, dt, 1e-12,
                                            dte if ratio == 10.0 else None))
        if ratio == 10.0:
            out = G.rkl2_advance("aniso", T, k, b, None, dt, s)
            for c in [(0, 0, 0), (3, 128, 511), (200, 60, 300)]:
                sub, idx, loc = W.subgrid(g, c, s + 2)
                Ts = _gather(T, idx)
                op = O.Operator(sub, O.spitzer_face_kappa(sub, Ts, cfg["kappa0"], cfg["T_cut"]), _gather(b, idx))
                ref = O.rkl2_advance(lambda x: (op.M @ x.ravel()).reshape(x.shape), Ts, dt, s)[loc]
                assert abs(float(out[c].item()) - ref) <= 1e-11 * abs(ref)
    s_list = [rec[r][0] for r in (10.0, 100.0, 1000.0)]
    it_list = [rec[r][1] for r in (10.0, 100.0, 1000.0)]
    assert s_list == sorted(s_list) and it_list == sorted(it_list), rec
    print("c3 sweep (ratio: stages, PCG iterations, full-grid residual):", rec)


@pytest.mark.parametrize("name", ["c1_spitzer64", "c2_visc64"])
def test_c1_c2_full_elementwise(dev, name):
    """BASELINE configs[1] / [2] at their full 64 x 64 x 128 size, element by element
    against the oracle: one RKL2 super-step (1e-11) and one BE + Jacobi-PCG step
    (iterations +-1; the GPU iterate meets the oracle system's own stopping test --
    a sparse direct solve for the exact answer is far too slow at this size)."""
    from paper_1610_01265_b200 import sts
    cfg = W.make_config(name)
    g = cfg["grid"]
    G = sts.Grid.from_grid(g)
    if name == "c1_spitzer64":
        ratio, mode = 100.0, "aniso"
        T = cfg["T"]
        kap = O.spitzer_face_kappa(g, T.numpy(), cfg["kappa0"], cfg["T_cut"])
        op = O.Operator(g, kap, cfg["b"].numpy())
        u, k, b, w = T, [torch.as_tensor(x) for x in kap], cfg["b"], None
        kd = G.face_kappa_spitzer(T.to(dev), cfg["kappa0"], cfg["T_cut"])
        for a, e in zip(kd, kap):
            np.testing.assert_allclose(a.cpu().numpy(), e, rtol=1e-13, atol=0)
    else:
        ratio, mode = 500.0, "iso"
        op = O.Operator(g, [f.numpy() for f in cfg["visc_faces"]], None, cfg["rho"].numpy())
        u, k, b, w = cfg["v"], cfg["visc_faces"], None, cfg["rho"]
    dte = O.dt_euler(op)
    dt = ratio * dte
    s = O.rkl2_num_stages(dt, dte)
    dv = lambda x: None if x is None else x.to(dev)  # noqa: E731
    kd = [x.to(dev) for x in k]
    assert abs(G.dt_euler(mode, kd, dv(b), dv(w)) - dte) <= 1e-12 * dte
    ref = O.rkl2_advance(lambda x: op.apply(x), u.numpy(), dt, s)
    out = G.rkl2_advance(mode, u.to(dev), kd, dv(b), dv(w), dt, s)
    d = out.cpu().numpy() - ref
    assert np.linalg.norm(d) <= 1e-11 * np.linalg.norm(ref)
    ref_be, it_ref = O.be_pcg_solve(op, u.numpy(), dt, rtol=1e-12)
    x, it = G.be_pcg_solve(mode, u.to(dev), kd, dv(b), dv(w), dt, 1e-12, 100000)
    assert all(abs(a - c) <= 1 for a, c in zip(it, it_ref)), (it, it_ref)
    A = O.be_system(op, dt).tocsr()
    D = A.diagonal()
    uu = u.numpy().reshape(-1, g.ncells)
    xx = x.cpu().numpy().reshape(uu.shape)
    for q in range(uu.shape[0]):
        bq = op.WV * uu[q]
        r = bq - A @ xx[q]
        # DESIGN R8 stopping test r.P^-1 r <= rtol^2 b.P^-1 b, with slack for the rounding
        # of the recurrence residual vs the true residual
        assert float(r @ (r / D)) <= (4e-12) ** 2 * float(bq @ (bq / D))
    assert np.linalg.norm(xx - ref_be.reshape(uu.shape)) <= 1e-9 * np.linalg.norm(ref_be)
    # fixed bar (north_star 1e-11): both solved to rtol 1e-15, where the iterate is pinned
    # to ~cond(A) 1e-15 (DESIGN R12)
    ref_fx, it_fx = O.be_pcg_solve(op, u.numpy(), dt, rtol=1e-15)
    x_fx, i_fx = G.be_pcg_solve(mode, u.to(dev), kd, dv(b), dv(w), dt, 1e-15, 100000)
    assert all(abs(a - c) <= 1 for a, c in zip(i_fx, it_fx)), (i_fx, it_fx)
    d_fx = np.linalg.norm(x_fx.cpu().numpy() - ref_fx) / np.linalg.norm(ref_fx)
    assert d_fx <= 1e-11, d_fx


def test_c1_lagged_conduction_rkl2_vs_be(dev):
    """BASELINE configs[1] at full size, 5 lagged-diffusivity steps at 100 dt_Euler
    with each method (face kappa recomputed from the current T every step):
    the two integrators of the same nonlinear problem agree to a few per cent (the
    paper's Sec. 6 validation, Fig. 10), and both conserve the volume-weighted total
    energy under the zero-flux walls to rounding."""
    from paper_1610_01265_b200 import sts
    cfg = W.make_config("c1_spitzer64", device=dev)
    g = cfg["grid"]
    G = sts.Grid.from_grid(g)
    b = cfg["b"]
    Tr, Tb = cfg["T"].clone(), cfg["T"].clone()
    geo = O.geometry(g)
    V = torch.as_tensor(geo["V"], device=dev)
    E0 = float((V * cfg["T"]).sum())
    dt = None
    for _ in range(5):
        kr = G.face_kappa_spitzer(Tr, cfg["kappa0"], cfg["T_cut"])
        kb = G.face_kappa_spitzer(Tb, cfg["kappa0"], cfg["T_cut"])
        dte = G.dt_euler("aniso", kr, b)
        dt = 100.0 * dte if dt is None else dt
        Tr = G.rkl2_advance("aniso", Tr, kr, b, None, dt, sts.rkl2_num_stages(dt, dte))
        Tb, _ = G.be_pcg_solve("aniso", Tb, kb, b, None, dt, 1e-12, 100000)
    d = float((Tr - Tb).norm() / Tb.norm())
    assert d < 0.05, d
    assert abs(float((V * Tr).sum()) - E0) <= 1e-12 * E0
    assert abs(float((V * Tb).sum()) - E0) <= 1e-9 * E0
