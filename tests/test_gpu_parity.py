"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by
element on identical seeded inputs.

Tolerances (BASELINE north_star, DESIGN.md §3 "Parity bar"):
  * operator / face diffusivity / Gershgorin: FP64 rounding of a different
    summation order -> relative L2 <= 1e-12, max-norm <= 1e-11 * max|ref|
  * RKL2: relative L2 <= 1e-11 after one super-step, <= 1e-9 after 20
  * BE+PCG (rtol 1e-12): relative L2 <= 1e-11 (one step), iteration counts
    identical within +-1
Sizes span several 32 x 8 (phi x theta) tiles and r-chunks with ragged tails,
plus the degenerate shapes (single plane / row / column, periodic n3 = 1, 2).
"""
import math
import zlib

import numpy as np
import pytest
import torch

import workloads as W
from oracle import core as O

pytestmark = pytest.mark.gpu

# the fixed PCG parity bar (DESIGN R12): solved to rtol 1e-15, a residual-stopped
# iterate is pinned to ~cond(A) 1e-15 (cond(A) ~ 1 + 2 dt/dt_exp <= ~1e3 here) well under
# north_star's 1e-11, so GPU, oracle and direct solve must agree to 1e-11
RTOL_FIXED = 1e-15
PREMISE = 2.5e-12   # the oracle's rtol-1e-15 iterate lies within a quarter of the bar of the direct solve


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import __graft_entry__ as e
    e.build()
    return torch.device("cuda", 0)


def sts():
    from paper_1610_01265_b200 import sts as S
    return S


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def max_rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def cpu(t):
    return t.detach().cpu().numpy()


def sph(shape, r1=20.0, dr0=0.005, periodic=True):
    n1, n2, n3 = shape
    g = W.spherical_grid(n1, n2, n3, r1=r1, dr0=dr0)
    if not periodic:
        g = W.Grid("spherical", g.x1f, np.linspace(0.3, 2.8, n2 + 1), np.linspace(0.0, 1.5, n3 + 1), False)
    return g


SHAPES = [(1, 1, 1), (1, 5, 7), (3, 1, 40), (5, 9, 1), (4, 3, 2), (20, 19, 70), (17, 9, 33)]


def _inputs(g, rng, bkind):
    shape = g.shape
    u = torch.as_tensor(rng.normal(size=shape) + 3.0)
    k = [torch.as_tensor(rng.uniform(0.5, 2.0, shape)) for _ in range(3)]
    if bkind == "random":
        b = W.random_unit_b(g, seed=int(rng.integers(1 << 30)))
    else:
        b = W.tilted_dipole_b(g, 30.0)
    return u, k, b


# ---------------------------------------------------------------- A3
# (shape, periodic, virtual slabs): even n3 takes the two-column vectorised pass (phi
# wrap, walls, n3 = 2, slab halos), odd n3 the one-column pass
FK_CASES = [((20, 19, 70), True, 1), ((7, 5, 33), True, 1), ((6, 4, 2), True, 1), ((9, 8, 64), False, 1),
            ((13, 6, 66), True, 3), ((10, 3, 9), False, 2), ((300, 2, 4), True, 1)]


@pytest.mark.parametrize("recipe", ["corona", "tr", "tr_fc"])
@pytest.mark.parametrize("shape,periodic,nv", FK_CASES)
def test_face_kappa_parity(dev, recipe, shape, periodic, nv):
    g = sph(shape, periodic=periodic)
    T = W.corona_T(g, seed=3) if recipe == "corona" else W.tr_corona_T(g, seed=3)
    fc_w = 0.5 if recipe == "tr_fc" else 0.0
    G = sts().Grid.from_grid(g, n_virtual=nv)
    k = G.face_kappa_spitzer(T.to(dev), 1e-9, 5e5, 10.0, fc_w)
    ref = O.spitzer_face_kappa(g, T.numpy(), 1e-9, 5e5, 10.0, fc_w)
    for d in range(3):
        assert max_rel(cpu(k[d]), ref[d]) <= 1e-13, d


# ---------------------------------------------------------------- A1 / A2
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("kind", ["aniso_random", "aniso_dipole", "iso", "iso3_weighted", "cart_iso"])
def test_op_apply_parity(dev, shape, kind):
    rng = np.random.default_rng(zlib.crc32(repr((shape, kind)).encode()))
    if kind == "cart_iso":
        n1, n2, n3 = shape
        g = W.Grid("cartesian", np.cumsum(np.r_[0, rng.uniform(0.5, 1.5, n1)]),
                   np.cumsum(np.r_[0, rng.uniform(0.5, 1.5, n2)]), np.arange(n3 + 1) * 0.7, False)
    else:
        g = sph(shape, periodic=(shape[2] != 33))
    u, k, b = _inputs(g, rng, "random" if kind == "aniso_random" else "dipole")
    w = None
    mode = "aniso" if kind.startswith("aniso") else "iso"
    if kind == "iso3_weighted":
        u = torch.as_tensor(rng.normal(size=(3,) + g.shape))
        w = torch.as_tensor(rng.uniform(0.2, 5.0, g.shape))
    G = sts().Grid.from_grid(g)
    F = G.op_apply(mode, u.to(dev), [x.to(dev) for x in k], b.to(dev) if mode == "aniso" else None,
                   None if w is None else w.to(dev))
    op = O.Operator(g, [x.numpy() for x in k], b.numpy() if mode == "aniso" else None,
                    None if w is None else w.numpy())
    ref = op.apply(u.numpy())
    if np.max(np.abs(ref)) == 0.0:
        assert np.max(np.abs(cpu(F))) == 0.0
        return
    assert rel_l2(cpu(F), ref) <= 1e-12
    assert max_rel(cpu(F), ref) <= 1e-11


@pytest.mark.parametrize("shape", [(1, 1, 1), (3, 1, 40), (5, 9, 1), (4, 3, 2), (20, 19, 70), (17, 9, 33)])
@pytest.mark.parametrize("mode", ["aniso", "iso"])
def test_dt_euler_parity(dev, shape, mode):
    rng = np.random.default_rng(7)
    g = sph(shape, periodic=(shape[2] != 33))
    u, k, b = _inputs(g, rng, "random")
    w = torch.as_tensor(rng.uniform(0.2, 5.0, g.shape)) if mode == "iso" else None
    G = sts().Grid.from_grid(g)
    dt = G.dt_euler(mode, [x.to(dev) for x in k], b.to(dev) if mode == "aniso" else None,
                    None if w is None else w.to(dev))
    op = O.Operator(g, [x.numpy() for x in k], b.numpy() if mode == "aniso" else None,
                    None if w is None else w.numpy())
    ref = O.dt_euler(op)
    if math.isinf(ref):
        assert math.isinf(dt)
    else:
        assert abs(dt - ref) <= 1e-13 * ref


# ---------------------------------------------------------------- A6
def _oracle_rkl2_run(g, T0, cfg, ratio, nsteps, b):
    """Lagged-diffusivity loop: refresh kappa, dt_exp, s every step."""
    T = T0.copy()
    dt = None
    ss = []
    for _ in range(nsteps):
        kap = O.spitzer_face_kappa(g, T, cfg["kappa0"], cfg["T_cut"])
        op = O.Operator(g, kap, b)
        dte = O.dt_euler(op)
        dt = ratio * dte if dt is None else dt
        s = O.rkl2_num_stages(dt, dte)
        ss.append(s)
        T = O.rkl2_advance(lambda x: (op.M @ x.ravel()).reshape(x.shape), T, dt, s)
    return T, ss


def _gpu_rkl2_run(G, T0, cfg, ratio, nsteps, b, inplace=False):
    S = sts()
    T = T0.clone()
    dt = None
    ss = []
    for _ in range(nsteps):
        k = G.face_kappa_spitzer(T, cfg["kappa0"], cfg["T_cut"])
        dte = G.dt_euler("aniso", k, b)
        dt = ratio * dte if dt is None else dt
        s = S.rkl2_num_stages(dt, dte)
        ss.append(s)
        T = G.rkl2_advance("aniso", T, k, b, None, dt, s, out=T if inplace else None)
    return T, ss


@pytest.mark.parametrize("tma,deviation", [(True, True), (True, False), (False, False)])
@pytest.mark.parametrize("nsteps,tol", [(1, 1e-11), (20, 1e-9)])
def test_rkl2_spitzer_parity(dev, nsteps, tol, tma, deviation):
    """Fig. 2 on the lagged Spitzer operator: TMA kernels with the stages in deviation
    form (default) or as printed, and the cp.async kernels."""
    cfg = W.make_config("c1_spitzer64", shape=(20, 19, 70))
    g = cfg["grid"]
    ref, s_ref = _oracle_rkl2_run(g, cfg["T"].numpy(), cfg, 100.0, nsteps, cfg["b"].numpy())
    G = sts().Grid.from_grid(g)
    G.set_tma(tma)
    G.set_rkl2_deviation(deviation)
    out, s_gpu = _gpu_rkl2_run(G, cfg["T"].to(dev), cfg, 100.0, nsteps, cfg["b"].to(dev))
    assert s_gpu == s_ref
    assert rel_l2(cpu(out), ref) <= tol


def test_rkl2_config0_parity(dev):
    cfg = W.make_config("c0_heat32")
    g = cfg["grid"]
    k = [f.numpy() for f in cfg["faces"]]
    op = O.Operator(g, k)
    dte = O.dt_euler(op)
    dt = 50.0 * dte
    s = O.rkl2_num_stages(dt, dte)
    G = sts().Grid.from_grid(g)
    kd = [f.to(dev) for f in cfg["faces"]]
    assert abs(G.dt_euler("iso", kd) - dte) <= 1e-15 * dte
    u_ref = cfg["u"].numpy()
    u = cfg["u"].to(dev)
    for n in range(10):
        u_ref = O.rkl2_advance(lambda x: (op.M @ x.ravel()).reshape(x.shape), u_ref, dt, s)
        u = G.rkl2_advance("iso", u, kd, None, None, dt, s)
        if n == 0:
            assert rel_l2(cpu(u), u_ref) <= 1e-11
    assert rel_l2(cpu(u), u_ref) <= 1e-9
    # conservation of the volume-weighted total (zero-flux walls): uniform V -> plain sum
    assert abs(float(u.sum()) - float(cfg["u"].sum())) <= 1e-12 * float(cfg["u"].abs().sum())


@pytest.mark.parametrize("deviation", [True, False])
def test_rkl2_viscosity_parity(dev, deviation):
    cfg = W.make_config("c2_visc64", shape=(20, 19, 70))
    g = cfg["grid"]
    k = [f.numpy() for f in cfg["visc_faces"]]
    op = O.Operator(g, k, None, cfg["rho"].numpy())
    dte = O.dt_euler(op)
    dt = 500.0 * dte
    s = O.rkl2_num_stages(dt, dte)
    ref = O.rkl2_advance(lambda x: op.apply(x), cfg["v"].numpy(), dt, s)
    G = sts().Grid.from_grid(g)
    G.set_rkl2_deviation(deviation)
    kd = [f.to(dev) for f in cfg["visc_faces"]]
    rho = cfg["rho"].to(dev)
    assert abs(G.dt_euler("iso", kd, None, rho) - dte) <= 1e-13 * dte
    out = G.rkl2_advance("iso", cfg["v"].to(dev), kd, None, rho, dt, s)
    assert rel_l2(cpu(out), ref) <= 1e-11


def test_rkl2_inplace_and_host_pointers(dev):
    cfg = W.make_config("c1_spitzer64", shape=(9, 17, 40))
    g = cfg["grid"]
    G = sts().Grid.from_grid(g)
    T = cfg["T"].to(dev)
    b = cfg["b"].to(dev)
    k = G.face_kappa_spitzer(T, cfg["kappa0"], cfg["T_cut"])
    dte = G.dt_euler("aniso", k, b)
    s = sts().rkl2_num_stages(30 * dte, dte)
    ref = G.rkl2_advance("aniso", T, k, b, None, 30 * dte, s)
    T2 = T.clone()
    G.rkl2_advance("aniso", T2, k, b, None, 30 * dte, s, out=T2)           # device in place
    assert torch.equal(T2, ref)
    Th = cfg["T"].clone().pin_memory()
    kh = [x.cpu() for x in k]
    out = G.rkl2_advance("aniso", Th, kh, b.cpu(), None, 30 * dte, s)       # host arrays (e2e path)
    assert torch.equal(out, ref.cpu())
    Th2 = cfg["T"].clone()                                                  # pageable, in place
    G.rkl2_advance("aniso", Th2, kh, b.cpu(), None, 30 * dte, s, out=Th2)
    assert torch.equal(Th2, ref.cpu())


# ---------------------------------------------------------------- A7
@pytest.mark.parametrize("case", ["c0", "c0_twopass", "c1", "c1_cpasync", "c1_nograph", "c1_twopass", "c2",
                                  "c2_nograph", "c2_twopass", "c2_twopass_nograph"])
def test_be_pcg_parity(dev, case):
    """BE + Jacobi-PCG vs the oracle (Fig. 1): merged one-pass iteration (default),
    the two-pass S / U iteration, the cp.async kernels, with and without graphs."""
    if case.startswith("c0"):
        cfg = W.make_config("c0_heat32")
        g = cfg["grid"]
        k, b, w, u, mode, ratio = cfg["faces"], None, None, cfg["u"], "iso", 50.0
    elif case.startswith("c1"):
        cfg = W.make_config("c1_spitzer64", shape=(20, 19, 70))
        g = cfg["grid"]
        k = [torch.as_tensor(x) for x in O.spitzer_face_kappa(g, cfg["T"].numpy(), cfg["kappa0"], cfg["T_cut"])]
        b, w, u, mode, ratio = cfg["b"], None, cfg["T"], "aniso", 100.0
    else:
        cfg = W.make_config("c2_visc64", shape=(20, 19, 70))
        g = cfg["grid"]
        k, b, w, u, mode, ratio = cfg["visc_faces"], None, cfg["rho"], cfg["v"], "iso", 500.0
    op = O.Operator(g, [x.numpy() for x in k], None if b is None else b.numpy(), None if w is None else w.numpy())
    dt = ratio * O.dt_euler(op)
    ref, it_ref = O.be_pcg_solve(op, u.numpy(), dt, rtol=1e-12)
    G = sts().Grid.from_grid(g)
    G.set_tma(case != "c1_cpasync")
    G.set_graphs(not case.endswith("nograph"))
    G.set_pcg_merged("twopass" not in case)
    out, it = G.be_pcg_solve(mode, u.to(dev), [x.to(dev) for x in k], None if b is None else b.to(dev),
                             None if w is None else w.to(dev), dt, 1e-12, 100000)
    assert all(abs(a - c) <= 1 for a, c in zip(it, it_ref)), (it, it_ref)
    assert rel_l2(cpu(out), ref) <= 1e-11
    # fixed bar: rtol 1e-15 against the direct solve and the oracle's rtol-1e-15 iterate
    import scipy.sparse.linalg as spl
    A = O.be_system(op, dt).tocsc()
    un = u.numpy().reshape(-1, g.ncells)
    exact = np.stack([spl.spsolve(A, op.WV * x) for x in un]).reshape(u.shape)
    ref_fx, it_fx = O.be_pcg_solve(op, u.numpy(), dt, rtol=RTOL_FIXED)
    out14, i_fx = G.be_pcg_solve(mode, u.to(dev), [x.to(dev) for x in k], None if b is None else b.to(dev),
                                None if w is None else w.to(dev), dt, RTOL_FIXED, 100000)
    assert all(abs(a - c) <= 1 for a, c in zip(i_fx, it_fx)), (i_fx, it_fx)
    assert rel_l2(cpu(out14), exact) <= 1e-11
    assert rel_l2(cpu(out14), ref_fx) <= 1e-11


def test_be_pcg_20_steps_parity(dev):
    """north_star: <= 1e-9 after 20 steps -- 20 lagged-diffusivity backward-Euler steps of
    the Spitzer problem (face kappa from the current T every step; dt =
    100 dt_exp of the first step) solved by Jacobi-PCG at rtol 1e-15, GPU vs oracle, and 20
    steps of the weighted 3-component viscosity problem."""
    cfg = W.make_config("c1_spitzer64", shape=(20, 19, 70))
    g = cfg["grid"]
    b = cfg["b"].numpy()
    G = sts().Grid.from_grid(g)
    bd = cfg["b"].to(dev)
    T_o, T_g = cfg["T"].numpy(), cfg["T"].to(dev)
    dt = None
    for n in range(20):
        kap = O.spitzer_face_kappa(g, T_o, cfg["kappa0"], cfg["T_cut"])
        op = O.Operator(g, kap, b)
        dt = 100.0 * O.dt_euler(op) if dt is None else dt
        T_o, it_o = O.be_pcg_solve(op, T_o, dt, rtol=RTOL_FIXED)
        kd = G.face_kappa_spitzer(T_g, cfg["kappa0"], cfg["T_cut"])
        T_g, it_g = G.be_pcg_solve("aniso", T_g, kd, bd, None, dt, RTOL_FIXED, 100000)
        assert abs(it_g[0] - it_o[0]) <= 1, (n, it_g, it_o)
        if n == 0:
            assert rel_l2(cpu(T_g), T_o) <= 1e-11
    assert rel_l2(cpu(T_g), T_o) <= 1e-9
    print("BE 20 steps, Spitzer: rel L2 =", rel_l2(cpu(T_g), T_o))
    cv = W.make_config("c2_visc64", shape=(20, 19, 70))
    opv = O.Operator(cv["grid"], [f.numpy() for f in cv["visc_faces"]], None, cv["rho"].numpy())
    dtv = 500.0 * O.dt_euler(opv)
    Gv = sts().Grid.from_grid(cv["grid"])
    kv, rho = [f.to(dev) for f in cv["visc_faces"]], cv["rho"].to(dev)
    v_o, v_g = cv["v"].numpy(), cv["v"].to(dev)
    for n in range(20):
        v_o, _ = O.be_pcg_solve(opv, v_o, dtv, rtol=RTOL_FIXED)
        v_g, _ = Gv.be_pcg_solve("iso", v_g, kv, None, rho, dtv, RTOL_FIXED, 100000)
        if n == 0:
            assert rel_l2(cpu(v_g), v_o) <= 1e-11
    assert rel_l2(cpu(v_g), v_o) <= 1e-9
    print("BE 20 steps, viscosity: rel L2 =", rel_l2(cpu(v_g), v_o))


def test_be_pcg_degenerate(dev):
    cfg = W.make_config("c1_spitzer64", shape=(6, 5, 8))
    g = cfg["grid"]
    G = sts().Grid.from_grid(g)
    b = cfg["b"].to(dev)
    k = G.face_kappa_spitzer(cfg["T"].to(dev), cfg["kappa0"], cfg["T_cut"])
    c = torch.full(g.shape, 3.0, dtype=torch.float64, device=dev)     # L c = 0 -> 0 iterations
    out, it = G.be_pcg_solve("aniso", c, k, b, None, 1e-3, 1e-12, 100)
    assert it == [0] and torch.equal(out, c)
    out, it = G.be_pcg_solve("aniso", cfg["T"].to(dev), k, b, None, 0.0, 1e-12, 100)   # dt = 0
    assert it == [0] and torch.equal(out, cfg["T"].to(dev))
    T = cfg["T"].to(dev)
    out, it = G.be_pcg_solve("aniso", T, k, b, None, 1.0, 1e-12, 2, allow_not_converged=True)
    assert it == [2]


# ---------------------------------------------------------------- decomposition emulation
@pytest.mark.parametrize("overlap", [False, True])
@pytest.mark.parametrize("nv", [2, 3, 7])
def test_virtual_slabs_match_single_domain(dev, nv, overlap):
    """n_virtual r-slabs exchange boundary planes through halo buffers exactly
    like the multi-GPU path -- waited for (one launch per slab, the default) or
    overlapped with the interior planes (one-plane boundary launches); per-cell
    arithmetic is identical -> bitwise equal operator / RKL2, PCG within rounding of
    its dot products."""
    cfg = W.make_config("c1_spitzer64", shape=(21, 19, 70))
    g = cfg["grid"]
    G1 = sts().Grid.from_grid(g)
    Gv = sts().Grid.from_grid(g, n_virtual=nv)
    Gv.set_halo_overlap(overlap)
    T = cfg["T"].to(dev)
    b = cfg["b"].to(dev)
    k = G1.face_kappa_spitzer(T, cfg["kappa0"], cfg["T_cut"])
    assert all(torch.equal(x, y) for x, y in zip(k, Gv.face_kappa_spitzer(T, cfg["kappa0"], cfg["T_cut"])))
    assert torch.equal(G1.op_apply("aniso", T, k, b), Gv.op_apply("aniso", T, k, b))
    d1, dv = G1.dt_euler("aniso", k, b), Gv.dt_euler("aniso", k, b)
    assert d1 == dv
    s = sts().rkl2_num_stages(100 * d1, d1)
    assert torch.equal(G1.rkl2_advance("aniso", T, k, b, None, 100 * d1, s),
                       Gv.rkl2_advance("aniso", T, k, b, None, 100 * d1, s))
    x1, i1 = G1.be_pcg_solve("aniso", T, k, b, None, 100 * d1, 1e-12, 10000)
    xv, iv = Gv.be_pcg_solve("aniso", T, k, b, None, 100 * d1, 1e-12, 10000)
    assert abs(i1[0] - iv[0]) <= 1 and rel_l2(cpu(xv), cpu(x1)) <= 1e-12
    # viscosity (3 components, weighted)
    cv = W.make_config("c2_visc64", shape=(21, 19, 70))
    kv = [f.to(dev) for f in cv["visc_faces"]]
    rho, v = cv["rho"].to(dev), cv["v"].to(dev)
    assert torch.equal(G1.op_apply("iso", v, kv, None, rho), Gv.op_apply("iso", v, kv, None, rho))
    dv = G1.dt_euler("iso", kv, None, rho)
    sv = sts().rkl2_num_stages(300 * dv, dv)
    assert torch.equal(G1.rkl2_advance("iso", v, kv, None, rho, 300 * dv, sv),
                       Gv.rkl2_advance("iso", v, kv, None, rho, 300 * dv, sv))
    y1, j1 = G1.be_pcg_solve("iso", v, kv, None, rho, 300 * dv, 1e-12, 10000)
    yv, jv = Gv.be_pcg_solve("iso", v, kv, None, rho, 300 * dv, 1e-12, 10000)
    assert all(abs(a - b) <= 1 for a, b in zip(j1, jv)) and rel_l2(cpu(yv), cpu(y1)) <= 1e-12


# ---------------------------------------------------------------- TMA vs cp.async kernels
TMA_CASES = [((20, 19, 70), True, 1), ((13, 17, 64), False, 1), ((5, 9, 2), True, 1), ((9, 16, 96), True, 1),
             ((21, 19, 62), True, 3), ((12, 8, 40), False, 2), ((7, 23, 33), True, 1)]


@pytest.mark.parametrize("shape,periodic,nv", TMA_CASES)
def test_tma_kernels_match_oracle_and_cpasync(dev, shape, periodic, nv):
    """The TMA + mbarrier pipelined kernels (even n3) and the cp.async kernels
    (forced, or odd n3) against the oracle: RKL2 super-step and BE+PCG, with
    periodic wrap tiles, non-periodic walls, several phi tiles and r chunks,
    and virtual r-slabs reading halo planes."""
    g = sph(shape, periodic=periodic)
    rng = np.random.default_rng(zlib.crc32(repr((shape, periodic, nv)).encode()))
    T = torch.as_tensor(1.5e6 * (1.0 + 0.3 * rng.uniform(-1, 1, g.shape)))
    b = W.random_unit_b(g, seed=int(rng.integers(1 << 30)))
    kap = O.spitzer_face_kappa(g, T.numpy(), 1e-9, 5e5)
    op = O.Operator(g, kap, b.numpy())
    dte = O.dt_euler(op)
    dt = 60.0 * dte
    s = O.rkl2_num_stages(dt, dte)
    ref = O.rkl2_advance(lambda x: (op.M @ x.ravel()).reshape(x.shape), T.numpy(), dt, s)
    ref_be, it_ref = O.be_pcg_solve(op, T.numpy(), dt, rtol=1e-12)
    ref_fx, it_fx = O.be_pcg_solve(op, T.numpy(), dt, rtol=RTOL_FIXED)
    # PCG stops on a residual, so its iterate is unique only to ~cond(A) * rtol: the GPU
    # iterate must be as close to the oracle's as the oracle's is to the exact solve
    import scipy.sparse.linalg as spl
    exact = spl.spsolve(O.be_system(op, dt).tocsc(), op.WV * T.numpy().ravel()).reshape(g.shape)
    tol_be = max(1e-11, rel_l2(ref_be, exact))
    print(f"R12 fallback bar at rtol 1e-12: tol_be = {tol_be:.2e}")
    print(f"fixed bar premise: oracle at rtol {RTOL_FIXED:g} vs direct solve {rel_l2(ref_fx, exact):.2e}")
    assert rel_l2(ref_fx, exact) <= PREMISE
    k = [torch.as_tensor(x).to(dev) for x in kap]
    outs = {}
    for tma, merged in ((True, True), (True, False), (False, False)):
        G = sts().Grid.from_grid(g, n_virtual=nv)
        G.set_tma(tma)
        G.set_pcg_merged(merged)
        u = G.rkl2_advance("aniso", T.to(dev), k, b.to(dev), None, dt, s)
        x, it = G.be_pcg_solve("aniso", T.to(dev), k, b.to(dev), None, dt, 1e-12, 10000)
        assert rel_l2(cpu(u), ref) <= 1e-11, tma
        # fixed bar (north_star 1e-11): at rtol 1e-15 the GPU iterate is within 1e-11 of
        # the direct solve and of the oracle's rtol-1e-15 iterate, iterations +-1
        x_fx, i_fx = G.be_pcg_solve("aniso", T.to(dev), k, b.to(dev), None, dt, RTOL_FIXED, 10000)
        assert rel_l2(cpu(x_fx), exact) <= 1e-11, (tma, merged, rel_l2(cpu(x_fx), exact))
        assert rel_l2(cpu(x_fx), ref_fx) <= 1e-11, (tma, merged)
        assert abs(i_fx[0] - it_fx[0]) <= 1, (tma, merged, i_fx, it_fx)
        # DESIGN R12: both residual-stopped iterates lie within tol_be of the direct solve
        assert rel_l2(cpu(x), exact) <= 2 * tol_be, (tma, merged)
        assert rel_l2(cpu(x), ref_be) <= 2 * tol_be, (tma, merged)
        assert abs(it[0] - it_ref[0]) <= 1, (tma, merged, it, it_ref)
        outs[(tma, merged)] = (cpu(u), cpu(x))
    assert rel_l2(outs[(True, True)][0], outs[(False, False)][0]) <= 1e-13
    for key in ((True, True), (True, False)):
        assert rel_l2(outs[key][1], outs[(False, False)][1]) <= 2 * tol_be   # all within tol_be of the oracle


ISO_CASES = [((20, 19, 70), True, 1, 3), ((13, 17, 64), False, 1, 3), ((5, 9, 2), True, 1, 2), ((9, 16, 96), True, 1, 1),
             ((21, 19, 62), True, 3, 3), ((12, 8, 40), False, 2, 2), ((7, 23, 33), True, 1, 3),
             # the 3-component merged pass's 13-row tile: one partial tile row, n3 = 2, and
             # virtual slabs of 2, 1, 1 planes
             ((6, 5, 8), True, 1, 3), ((5, 9, 2), True, 2, 3), ((4, 11, 16), False, 3, 3)]


@pytest.mark.parametrize("shape,periodic,nv,nc", ISO_CASES)
def test_iso_tma_kernels_match_oracle_and_cpasync(dev, shape, periodic, nv, nc):
    """Isotropic weighted (viscosity-type) operator, 1-3 components: warp-specialised
    TMA kernels (even n3) vs cp.async kernels vs the oracle, RKL2 and BE+PCG."""
    g = sph(shape, periodic=periodic)
    rng = np.random.default_rng(zlib.crc32(repr(("iso", shape, periodic, nv, nc)).encode()))
    k = [rng.uniform(0.5, 2.0, g.shape) for _ in range(3)]
    w = rng.uniform(0.5, 2.0, g.shape)
    v = rng.normal(size=(nc,) + g.shape)
    op = O.Operator(g, k, None, w)
    dte = O.dt_euler(op)
    dt = 200.0 * dte
    s = O.rkl2_num_stages(dt, dte)
    ref = O.rkl2_advance(op.apply, v, dt, s)
    ref_be, it_ref = O.be_pcg_solve(op, v, dt, rtol=1e-12)
    ref_fx, it_fx = O.be_pcg_solve(op, v, dt, rtol=RTOL_FIXED)
    import scipy.sparse.linalg as spl
    A = O.be_system(op, dt).tocsc()
    exact = np.stack([spl.spsolve(A, op.WV * x.ravel()).reshape(g.shape) for x in v])
    tol_be = max(1e-11, rel_l2(ref_be, exact))
    print(f"R12 fallback bar at rtol 1e-12: tol_be = {tol_be:.2e}")
    print(f"fixed bar premise: oracle at rtol {RTOL_FIXED:g} vs direct solve {rel_l2(ref_fx, exact):.2e}")
    assert rel_l2(ref_fx, exact) <= PREMISE
    kd = [torch.as_tensor(x).to(dev) for x in k]
    wd = torch.as_tensor(w).to(dev)
    vd = torch.as_tensor(v).to(dev)
    if nc == 1:
        vd = vd[0].contiguous()
    outs = {}
    for tma, merged in ((True, True), (True, False), (False, False)):
        G = sts().Grid.from_grid(g, n_virtual=nv)
        G.set_tma(tma)
        G.set_pcg_merged(merged)
        F = G.op_apply("iso", vd, kd, None, wd)
        assert rel_l2(cpu(F).reshape(v.shape), op.apply(v)) <= 1e-12, tma
        u = G.rkl2_advance("iso", vd, kd, None, wd, dt, s)
        x, it = G.be_pcg_solve("iso", vd, kd, None, wd, dt, 1e-12, 10000)
        assert rel_l2(cpu(u).reshape(v.shape), ref) <= 1e-11, tma
        x_fx, i_fx = G.be_pcg_solve("iso", vd, kd, None, wd, dt, RTOL_FIXED, 10000)
        assert rel_l2(cpu(x_fx).reshape(v.shape), exact) <= 1e-11, (tma, merged)
        assert rel_l2(cpu(x_fx).reshape(v.shape), ref_fx) <= 1e-11, (tma, merged)
        assert all(abs(a - b) <= 1 for a, b in zip(i_fx, it_fx)), (tma, merged, i_fx, it_fx)
        # DESIGN R12: both residual-stopped iterates lie within tol_be of the direct solve
        assert rel_l2(cpu(x).reshape(v.shape), exact) <= 2 * tol_be, (tma, merged)
        assert rel_l2(cpu(x).reshape(v.shape), ref_be) <= 2 * tol_be, (tma, merged)
        assert all(abs(a - b) <= 1 for a, b in zip(it, it_ref)), (tma, merged, it, it_ref)
        outs[(tma, merged)] = (cpu(u), cpu(x))
    assert rel_l2(outs[(True, True)][0], outs[(False, False)][0]) <= 1e-13
    for key in ((True, True), (True, False)):
        assert rel_l2(outs[key][1], outs[(False, False)][1]) <= 2 * tol_be   # all within tol_be of the oracle


@pytest.mark.parametrize("merged", [True, False])
@pytest.mark.parametrize("nv", [1, 3])
@pytest.mark.parametrize("mode", ["aniso", "iso"])
def test_pcg_graph_replay_is_bitwise_identical(dev, nv, mode, merged):
    """CUDA-graph replay of iteration pairs (incl. the virtual-slab fork/join of the
    halo exchange inside the graph) runs exactly the kernels of direct launches."""
    cfg = W.make_config("c1_spitzer64" if mode == "aniso" else "c2_visc64", shape=(21, 19, 70))
    g = cfg["grid"]
    outs = []
    for graphs in (True, False):
        G = sts().Grid.from_grid(g, n_virtual=nv)
        G.set_graphs(graphs)
        G.set_pcg_merged(merged)
        if mode == "aniso":
            T, b = cfg["T"].to(dev), cfg["b"].to(dev)
            k = G.face_kappa_spitzer(T, cfg["kappa0"], cfg["T_cut"])
            dte = G.dt_euler("aniso", k, b)
            x, it = G.be_pcg_solve("aniso", T, k, b, None, 100 * dte, 1e-12, 10000)
        else:
            kv = [f.to(dev) for f in cfg["visc_faces"]]
            rho, v = cfg["rho"].to(dev), cfg["v"].to(dev)
            dte = G.dt_euler("iso", kv, None, rho)
            x, it = G.be_pcg_solve("iso", v, kv, None, rho, 500 * dte, 1e-12, 10000)
        outs.append((x.clone(), it))
    assert outs[0][1] == outs[1][1]
    assert torch.equal(outs[0][0], outs[1][0])


def test_smoke_entry(dev):
    import __graft_entry__ as e
    e.smoke()


# ---------------------------------------------------------------- A8 (PAPER.md:341 remedies)
@pytest.mark.parametrize("frac,n_sub,tma", [(0.25, 1, True), (0.25, 2, False), (0.0, 3, True), (0.5, 1, True)])
def test_rkl2_hybrid_parity(dev, frac, n_sub, tma):
    cfg = W.make_config("c1_spitzer64", shape=(20, 19, 70))
    g = cfg["grid"]
    kap = O.spitzer_face_kappa(g, cfg["T"].numpy(), cfg["kappa0"], cfg["T_cut"])
    op = O.Operator(g, kap, cfg["b"].numpy())
    dte = O.dt_euler(op)
    dt = 100.0 * dte
    n_euler = 0 if frac == 0 else int(math.ceil(frac * dt / (0.5 * dte) - 1e-12))
    ref, s_ref = O.rkl2_hybrid_advance(lambda x: (op.M @ x.ravel()).reshape(x.shape), cfg["T"].numpy(), dt, dte,
                                       frac, n_euler, n_sub)
    G = sts().Grid.from_grid(g)
    G.set_tma(tma)
    out, (ne, s) = G.rkl2_advance_hybrid("aniso", cfg["T"].to(dev), [torch.as_tensor(x).to(dev) for x in kap],
                                         cfg["b"].to(dev), None, dt, dte, frac, None, n_sub)
    assert ne == n_euler and s == s_ref
    assert rel_l2(cpu(out), ref) <= 1e-11
    # viscosity (3 components, weighted) through the same entry point
    cv = W.make_config("c2_visc64", shape=(12, 9, 40))
    opv = O.Operator(cv["grid"], [f.numpy() for f in cv["visc_faces"]], None, cv["rho"].numpy())
    dtev = O.dt_euler(opv)
    ne_v = 0 if frac == 0 else int(math.ceil(frac * 50 * dtev / (0.5 * dtev) - 1e-12))
    refv, _ = O.rkl2_hybrid_advance(opv.apply, cv["v"].numpy(), 50 * dtev, dtev, frac, ne_v, n_sub)
    Gv = sts().Grid.from_grid(cv["grid"])
    outv, _ = Gv.rkl2_advance_hybrid("iso", cv["v"].to(dev), [f.to(dev) for f in cv["visc_faces"]], None,
                                     cv["rho"].to(dev), 50 * dtev, dtev, frac, None, n_sub)
    assert rel_l2(cpu(outv), refv) <= 1e-11


@pytest.mark.parametrize("merged", [True, False])
@pytest.mark.parametrize("graphs", [True, False])
def test_communication_profile_matches_paper(dev, graphs, merged):
    """PAPER.md Sec. 2.4 / Figs. 1-2 boxed terms: an RKL2 super-step needs s neighbour
    exchanges and no global reduction; BE+PCG needs one exchange per matvec (+1 for the
    initial residual) and global reductions every iteration -- two (Fig. 1) in the
    two-pass iteration, one in the merged iteration -- counted on a decomposed
    (virtual-slab) grid, graph replay included."""
    cfg = W.make_config("c1_spitzer64", shape=(21, 19, 70))
    g = cfg["grid"]
    G = sts().Grid.from_grid(g, n_virtual=3)
    G.set_graphs(graphs)
    G.set_pcg_merged(merged)
    T, b = cfg["T"].to(dev), cfg["b"].to(dev)
    k = G.face_kappa_spitzer(T, cfg["kappa0"], cfg["T_cut"])
    dte = G.dt_euler("aniso", k, b)
    s = sts().rkl2_num_stages(100 * dte, dte)
    l0, g0 = G.comm_counts
    G.rkl2_advance("aniso", T, k, b, None, 100 * dte, s)
    l1, g1 = G.comm_counts
    assert (l1 - l0, g1 - g0) == (s, 0)
    _, it = G.be_pcg_solve("aniso", T, k, b, None, 100 * dte, 1e-12, 10000)
    l2, g2 = G.comm_counts
    # iterations launched in whole batches may overshoot convergence by a few no-op
    # passes (every kernel exits on the device-side done flag); those count as events
    n = (l2 - l1) - 1
    assert n >= it[0] and n - it[0] <= 64
    assert g2 - g1 == (1 if merged else 2) * n + 1
    G1 = sts().Grid.from_grid(g)                      # a single slab communicates nothing
    G1.rkl2_advance("aniso", T, k, b, None, 100 * dte, s)
    assert G1.comm_counts == (0, 0)


def test_host_pointer_paths_match_device(dev):
    """The C ABI accepts host arrays (the end-to-end path): every entry point stages
    them and returns the same results as with device arrays."""
    cfg = W.make_config("c1_spitzer64", shape=(9, 17, 40))
    g = cfg["grid"]
    G = sts().Grid.from_grid(g)
    T, b = cfg["T"].to(dev), cfg["b"].to(dev)
    k = G.face_kappa_spitzer(T, cfg["kappa0"], cfg["T_cut"])
    kh = G.face_kappa_spitzer(cfg["T"].clone(), cfg["kappa0"], cfg["T_cut"])
    assert all(torch.equal(a.cpu(), c) for a, c in zip(k, kh))
    dte = G.dt_euler("aniso", k, b)
    assert G.dt_euler("aniso", [x.cpu() for x in k], b.cpu()) == dte
    F = G.op_apply("aniso", T, k, b)
    assert torch.equal(G.op_apply("aniso", cfg["T"].clone(), [x.cpu() for x in k], b.cpu()), F.cpu())
    x, it = G.be_pcg_solve("aniso", T, k, b, None, 50 * dte, 1e-12, 10000)
    xh, ith = G.be_pcg_solve("aniso", cfg["T"].clone().pin_memory(), [x_.cpu() for x_ in k], b.cpu(), None,
                             50 * dte, 1e-12, 10000)
    assert ith == it and torch.equal(xh, x.cpu())
    u, st = G.rkl2_advance_hybrid("aniso", T, k, b, None, 50 * dte, dte, 0.25)
    uh, sth = G.rkl2_advance_hybrid("aniso", cfg["T"].clone(), [x_.cpu() for x_ in k], b.cpu(), None, 50 * dte,
                                    dte, 0.25)
    assert st == sth and torch.equal(uh, u.cpu())


def test_argument_errors_on_a_live_grid(dev):
    """Invalid calls return STS_ERR_* with a message and leave the handle usable."""
    S = sts()
    cfg = W.make_config("c1_spitzer64", shape=(6, 5, 8))
    G = S.Grid.from_grid(cfg["grid"])
    T, b = cfg["T"].to(dev), cfg["b"].to(dev)
    k = G.face_kappa_spitzer(T, cfg["kappa0"], cfg["T_cut"])
    with pytest.raises(S.StsError, match="s must be >= 2"):
        G.rkl2_advance("aniso", T, k, b, None, 1.0, 1)
    with pytest.raises(S.StsError, match="requires b"):
        G.rkl2_advance("aniso", T, k, None, None, 1.0, 3)
    with pytest.raises(S.StsError, match="ncomp"):
        G.op_apply("aniso", torch.stack([T, T]), k, b)
    with pytest.raises(S.StsError, match="kmax"):
        G.be_pcg_solve("aniso", T, k, b, None, 1.0, 1e-12, 0)
    with pytest.raises(S.StsError, match="alias"):
        G.op_apply("aniso", T, k, b, out=T)
    with pytest.raises(S.StsError, match="dt_exp"):
        G.rkl2_advance_hybrid("aniso", T, k, b, None, 10.0, 1.0, 0.5, n_euler=1)
    with pytest.raises(S.StsError, match="kmax reached"):
        G.be_pcg_solve("aniso", T, k, b, None, 1.0, 1e-12, 1)
    dte = G.dt_euler("aniso", k, b)                     # still usable
    assert math.isfinite(dte) and dte > 0


def test_pcg_breakdown_and_slab_state_errors(dev):
    """PCG breakdown (not SPD / non-finite input) returns STS_ERR_BREAKDOWN instead of
    carrying NaN alphas into x (Fig. 1 divides by p.A p); an r-slab handle
    used before sts_comm_init returns STS_ERR_STATE instead of reading outside the arrays."""
    S = sts()
    cfg = W.make_config("c2_visc64", shape=(8, 9, 16))
    g = cfg["grid"]
    kv = [f.to(dev) for f in cfg["visc_faces"]]
    v = cfg["v"].to(dev)
    for merged in (True, False):
        G = S.Grid.from_grid(g)
        G.set_pcg_merged(merged)
        neg = -cfg["rho"].to(dev)                         # w < 0: A = wV - dt L is negative definite
        with pytest.raises(S.StsError) as e:
            G.be_pcg_solve("iso", v, kv, None, neg, 1e-3, 1e-12, 1000)
        assert e.value.code == S.STS_ERR_BREAKDOWN and "breakdown" in str(e.value)
        bad = v.clone()
        bad[1, 3, 4, 5] = float("nan")
        with pytest.raises(S.StsError) as e:
            G.be_pcg_solve("iso", bad, kv, None, cfg["rho"].to(dev), 1e-3, 1e-12, 1000)
        assert e.value.code == S.STS_ERR_BREAKDOWN
        x, it = G.be_pcg_solve("iso", v, kv, None, cfg["rho"].to(dev), 1e-3, 1e-12, 1000)   # still usable
        assert all(i > 0 for i in it) and torch.isfinite(x).all()
    Gs = S.Grid.from_grid(g, i0=2, nl=3)                  # planes [2, 5) of 8: two neighbours
    w3 = W.r_slab(g, 2, 3)
    T = torch.ones(w3.shape, dtype=torch.float64, device=dev)
    k3 = [torch.ones_like(T) for _ in range(3)]
    with pytest.raises(S.StsError, match="sts_comm_init") as e:
        Gs.op_apply("iso", T, k3)
    assert e.value.code == -5
    with pytest.raises(S.StsError, match="sts_comm_init"):
        Gs.face_kappa_spitzer(T, 1e-9, 5e5)


@pytest.mark.parametrize("mode", ["aniso", "iso"])
def test_resident_coefficients_match_explicit(dev, mode):
    """Coefficients bound once (device arrays referenced, host arrays uploaded, face kappa
    written in place) give bit-identical results to passing the arrays every call, for
    every entry point; the derived data (vertex coefficients, folded face coefficients,
    Gershgorin bound) is rebuilt after a rebind."""
    S = sts()
    if mode == "aniso":
        cfg = W.make_config("c1_spitzer64", shape=(13, 17, 40))
        T, b = cfg["T"].to(dev), cfg["b"].to(dev)
        u, ratio, w = T, 100.0, None
    else:
        cfg = W.make_config("c2_visc64", shape=(13, 17, 40))
        u, b, w, ratio = cfg["v"].to(dev), None, cfg["rho"].to(dev), 500.0
    g = cfg["grid"]
    G = S.Grid.from_grid(g)
    Gr = S.Grid.from_grid(g)
    if mode == "aniso":
        k = G.face_kappa_spitzer(T, cfg["kappa0"], cfg["T_cut"])
        Gr.bind_coeffs("aniso", None, b=b.cpu().pin_memory())          # b from pinned host memory
        assert Gr.face_kappa_spitzer(T, cfg["kappa0"], cfg["T_cut"], resident=True) is None
    else:
        k = [f.to(dev) for f in cfg["visc_faces"]]
        Gr.bind_coeffs("iso", k, w=w.cpu())                             # w from pageable host memory
    dte = G.dt_euler(mode, k, b, w)
    assert Gr.dt_euler(mode, None) == dte and Gr.dt_euler(mode, None) == dte     # (cached)
    dt = ratio * dte
    s = S.rkl2_num_stages(dt, dte)
    assert torch.equal(G.op_apply(mode, u, k, b, w), Gr.op_apply(mode, u, None))
    assert torch.equal(G.rkl2_advance(mode, u, k, b, w, dt, s), Gr.rkl2_advance(mode, u, None, dt=dt, s=s))
    x1, i1 = G.be_pcg_solve(mode, u, k, b, w, dt, 1e-12, 10000)
    x2, i2 = Gr.be_pcg_solve(mode, u, None, dt=dt, rtol=1e-12, kmax=10000)
    assert i1 == i2 and torch.equal(x1, x2)
    # rebind different coefficients: the derived data follows
    k2 = [x * 1.5 for x in k]
    Gr.bind_coeffs(mode, k2)
    assert Gr.dt_euler(mode, None) == G.dt_euler(mode, k2, b, w)
    assert torch.equal(G.op_apply(mode, u, k2, b, w), Gr.op_apply(mode, u, None))
    x3, i3 = Gr.be_pcg_solve(mode, u, None, dt=dt, rtol=1e-12, kmax=10000)
    x4, i4 = G.be_pcg_solve(mode, u, k2, b, w, dt, 1e-12, 10000)
    assert i3 == i4 and torch.equal(x3, x4)
    with pytest.raises(S.StsError, match="must be NULL"):
        Gr.op_apply(mode, u, None, b=b if b is not None else w)
    Gr.unbind_coeffs(mode)
    with pytest.raises(S.StsError, match="none are bound"):
        Gr.op_apply(mode, u, None)


def test_async_host_path_and_async_solve(dev):
    """The asynchronous host-array path (pinned arrays, outputs read after join +
    synchronize) and be_pcg_solve_async (iterations and status written when the stream
    reaches the end of the solve) return what the synchronous device path returns."""
    S = sts()
    cfg = W.make_config("c1_spitzer64", shape=(13, 17, 40))
    g = cfg["grid"]
    T, b = cfg["T"].to(dev), cfg["b"].to(dev)
    G = S.Grid.from_grid(g)
    k = G.face_kappa_spitzer(T, cfg["kappa0"], cfg["T_cut"])
    dte = G.dt_euler("aniso", k, b)
    s = S.rkl2_num_stages(100 * dte, dte)
    ref_rk = G.rkl2_advance("aniso", T, k, b, None, 100 * dte, s)
    ref_be, ref_it = G.be_pcg_solve("aniso", T, k, b, None, 100 * dte, 1e-12, 10000)
    Ga = S.Grid.from_grid(g)
    Ga.async_host = True
    Ga.bind_coeffs("aniso", [x.cpu().pin_memory() for x in k], b.cpu().pin_memory())
    Th = cfg["T"].clone().pin_memory()
    outs = []
    for rep in range(3):                                   # staging buffers are reused across calls
        rk = Ga.rkl2_advance("aniso", Th, None, dt=100 * dte, s=s)
        be, res = Ga.be_pcg_solve_async("aniso", Th, None, dt=100 * dte, rtol=1e-12, kmax=10000)
        outs.append((rk, be, res))
    Ga.join()
    torch.cuda.synchronize()
    for rk, be, res in outs:
        assert torch.equal(rk, ref_rk.cpu()) and torch.equal(be, ref_be.cpu())
        assert res.iters == ref_it and res.status == 0
    # a device solve through the async entry point, stopped at kmax: status, not an exception
    x, res = G.be_pcg_solve_async("aniso", T, k, b, None, 100 * dte, 1e-12, 3)
    torch.cuda.synchronize()
    assert res.iters == [3] and res.status == S.STS_ERR_NOT_CONVERGED


@pytest.mark.parametrize("mode", ["aniso", "iso"])
@pytest.mark.parametrize("graphs", [True, False])
def test_nccl_one_rank_path_matches_single_process(dev, mode, graphs):
    """The NCCL path of the PCG solve (per-rank partial sums -> ncclAllReduce -> scalar
    kernel; host-polled batches; iteration pairs replayed from a captured graph with the
    NCCL calls inside) on a one-rank communicator equals the single-process path to the
    rounding of the dot-product summation order; RKL2 (no reductions) bit for bit."""
    S = sts()
    name = "c1_spitzer64" if mode == "aniso" else "c2_visc64"
    cfg = W.make_config(name, shape=(13, 17, 40))
    g = cfg["grid"]
    G1 = S.Grid.from_grid(g)
    Gn = S.Grid.from_grid(g)
    Gn.comm_init(1, 0, S.nccl_unique_id())
    Gn.set_graphs(graphs)
    if mode == "aniso":
        u, b, w = cfg["T"].to(dev), cfg["b"].to(dev), None
        k = G1.face_kappa_spitzer(u, cfg["kappa0"], cfg["T_cut"])
        ratio = 100.0
    else:
        u, b, w = cfg["v"].to(dev), None, cfg["rho"].to(dev)
        k = [f.to(dev) for f in cfg["visc_faces"]]
        ratio = 500.0
    dte = G1.dt_euler(mode, k, b, w)
    assert Gn.dt_euler(mode, k, b, w) == dte
    s = S.rkl2_num_stages(ratio * dte, dte)
    assert torch.equal(G1.rkl2_advance(mode, u, k, b, w, ratio * dte, s),
                       Gn.rkl2_advance(mode, u, k, b, w, ratio * dte, s))
    x1, i1 = G1.be_pcg_solve(mode, u, k, b, w, ratio * dte, 1e-12, 10000)
    l0 = Gn.kernel_launches
    xn, i_n = Gn.be_pcg_solve(mode, u, k, b, w, ratio * dte, 1e-12, 10000)
    assert all(abs(a - c) <= 1 for a, c in zip(i1, i_n)), (i1, i_n)
    assert rel_l2(cpu(xn), cpu(x1)) <= 1e-12
    # no more than a couple of no-op iterations after convergence (batches sized from the
    # observed rate): launches per iteration are bounded
    per_it = 4 if mode == "aniso" else 4
    assert Gn.kernel_launches - l0 <= per_it * (max(i_n) + 3) + 40


def test_host_path_pageable_and_virtual_slab_bindings(dev):
    """Pageable host arrays make a call synchronous (outputs written back on return, no
    join); resident bindings on a virtual-slab grid (binding work on the compute stream,
    halos of the coefficients exchanged every call) equal the single domain bit for bit;
    an asynchronous solve on host arrays in pageable memory falls back to synchronous."""
    S = sts()
    cfg = W.make_config("c1_spitzer64", shape=(13, 17, 40))
    g = cfg["grid"]
    T, b = cfg["T"].to(dev), cfg["b"].to(dev)
    G1 = S.Grid.from_grid(g)
    k = G1.face_kappa_spitzer(T, cfg["kappa0"], cfg["T_cut"])
    dte = G1.dt_euler("aniso", k, b)
    s = S.rkl2_num_stages(60 * dte, dte)
    ref = G1.rkl2_advance("aniso", T, k, b, None, 60 * dte, s)
    ref_x, ref_it = G1.be_pcg_solve("aniso", T, k, b, None, 60 * dte, 1e-12, 10000)
    Gp = S.Grid.from_grid(g)
    Gp.async_host = True                       # no join in the binding: pageable => synchronous
    Th, kh, bh = cfg["T"].clone(), [x.cpu() for x in k], cfg["b"].clone()
    assert not Th.is_pinned()
    out = torch.empty_like(Th)
    Gp.rkl2_advance("aniso", Th, kh, bh, None, 60 * dte, s, out=out)
    assert torch.equal(out, ref.cpu())
    xo = torch.empty_like(Th)
    _, res = Gp.be_pcg_solve_async("aniso", Th, kh, bh, None, 60 * dte, 1e-12, 10000, out=xo)
    assert res.status == 0 and res.iters == ref_it and torch.equal(xo, ref_x.cpu())
    for nv in (1, 3):
        Gv = S.Grid.from_grid(g, n_virtual=nv)
        Gv.bind_coeffs("aniso", None, b=b)
        Gv.face_kappa_spitzer(T, cfg["kappa0"], cfg["T_cut"], resident=True)
        assert Gv.dt_euler("aniso", None) == dte
        assert torch.equal(Gv.rkl2_advance("aniso", T, None, dt=60 * dte, s=s), ref)
        xv, iv = Gv.be_pcg_solve("aniso", T, None, dt=60 * dte, rtol=1e-12, kmax=10000)
        assert abs(iv[0] - ref_it[0]) <= 1 and rel_l2(cpu(xv), cpu(ref_x)) <= 1e-12
