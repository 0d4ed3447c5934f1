#!/usr/bin/env python3
"""bench.py — Gcell-updates/s of the B200 RKL2 / BE+Jacobi-PCG parabolic advance.

One *step* = one pass of the whole hot path (DESIGN.md §0 rows A1-A7) over the
BASELINE.json configs[4] workload (Spitzer conduction + viscosity on the
512 x 512 x 1024 spherical grid, FP64, dt = 300 dt_exp):
  conduction: lagged face kappa -> Gershgorin dt_exp -> s -> RKL2 super-step,
              and BE solved by Jacobi-PCG (rtol 1e-12)
  viscosity : Gershgorin dt_exp -> s -> RKL2 super-step (3 components),
              and BE solved by Jacobi-PCG (3 components)
every step advancing the same resident inputs (deterministic work per step).
A cell-update is one cell advanced by one RKL2 stage or one PCG iteration
(a 3-component velocity cell counts once; the vector PCG counts its slowest
component).  value = total cell-updates of all ranks / max-over-ranks device time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...      (r-slab decomposition, NCCL)
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402

METRIC = "Gcell-updates/s per RKL2 stage and PCG iter (1/2/4/8 B200), % HBM roofline"
UNIT = "Gcell-updates/s"
RATIO = {"c1_spitzer64": 100.0, "c2_visc64": 500.0, "c3_spitzer256": 100.0, "c4_scale512": 300.0}
RTOL = 1e-12
KMAX = 50000
# bounded CPU sample of the same workload for the oracle baseline (cells of the box)
CPU_BOX = (12, 40, 64)


# classes whose HBM fraction is not their bound (DESIGN.md §5.3 / §5.4)
KERNEL_NOTES = {
    "aniso_gersh": "bound by its FP64 / shared-memory work (~115 FP64 instructions per cell for the 27 "
                   "|L_ij| of a row), not by HBM; once per step",
    "pcg_reduce": "one 1024-thread block per PCG iteration: launch-latency bound, no HBM traffic",
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ----------------------------------------------------------------------------
# algorithmic HBM bytes per cell for each kernel class: every
# field read or written exactly once, FP64
# ----------------------------------------------------------------------------
def bytes_per_cell(kind, ncomp=1, active=None, first=False):
    c = ncomp if active is None else active
    table = {
        "face_kappa": 8 + 24,
        # anisotropic passes stream u + the 3 frozen vertex coefficients e
        "vertex_coef": 48 + 24,
        "aniso_F": 8 + 24 + 8,
        "aniso_rkl2_first": 8 + 24 + 16,
        "aniso_rkl2_stage": 8 + 24 + 24 + 8,
        "aniso_pcg_r0": 8 + 24 + 32,          # TMA R0: u, e in; r, x, z, d out
        "aniso_pcg_ap": 8 + 24 + 8,
        # fused S-pass: z, pold, x, e in; p, y, x out (first iteration: z, e in; p, y out)
        "aniso_pcg_s": (8 + 24 + 16) if first else (24 + 24 + 24),
        "aniso_gersh": 24,                   # row sums from the frozen vertex coefficients e
        "iso_rkl2_first": 8 * c + 32 + 16 * c,
        "iso_rkl2_stage": 32 * c + 32 + 8 * c,
        "iso_pcg_r0": 8 * c + 32 + 16 * c + 8,     # fused path: r, x, d (no z)
        "iso_pcg_ap": 16 * c + 32,
        # fused S-pass: r, pold, x (+ d, k1, k2, k3, w) in; p, y, x out (first: r, d in; p, y out);
        # z = r d is formed in the pass, never stored
        "iso_pcg_s": (24 * c + 40) if first else (48 * c + 40),
        # U-pass of the isotropic fused path: r, y, d in; r out (no z)
        "pcg_update_noz": 24 * c + 8,
        "iso_gersh": 32,
        # U-pass: r, y, d in; r, z out
        "pcg_update": 32 * c + 8,
        # p pass of the unfused S-pass: z, pold, x in; p, x out (first: z in, p out)
        "pcg_pupdate": 16 * c if first else 40 * c,
        "pcg_xfinal": 24 * c,
        # merged iteration (one pass): p_{k-2}, w_{k-1}, p_{k-1}, x (+ e, d) in; p, w, x out
        # (first: z0 (+ e, d) in; p, w out); z is never stored; R0 of the merged path writes z0
        "aniso_pcg_m": (8 + 24 + 8 + 16) if first else (32 + 24 + 8 + 24),
        # (the isotropic pass recomputes d from the staged face coefficients)
        "iso_pcg_m": (24 * c + 32) if first else (56 * c + 32),
        "iso_pcg_r0_m": 8 * c + 32 + 24 * c + 8,
        # RKL2 stage in deviation form (D_j = Y_j - Y0): D_{j-1}, D_{j-2}, M0 (+ e / k, w) in; D_j out
        "aniso_rkl2_dstage": 8 + 24 + 16 + 8,
        "iso_rkl2_dstage": 24 * c + 32 + 8 * c,
    }
    return table[kind]


def algorithmic_bytes(ncells, s_c, it_c, s_v, it_v, fused_c=True, fused_v=False, merged_c=False, merged_v=False,
                      dev_c=False, dev_v=False, xm_c=None, xm_v=None):
    """Total algorithmic bytes per class for one step on `ncells` local cells.
    xm_c / xm_v: (skipped, caught_up) x-update passes per component of the merged PCG
    solves (DESIGN.md §5.3 "x in pairs"): a skipped pass moves 16 B/cell/component less
    (no x read / write); a catch-up pass moves what a normal pass does (its own z_{k-1}
    is staged)."""
    B = {}
    add = lambda k, v: B.__setitem__(k, B.get(k, 0.0) + v * ncells)  # noqa: E731
    if s_c:
        _cond_bytes(add, s_c, it_c, fused_c, merged_c, dev_c)
        if merged_c and xm_c:
            add("aniso_pcg_m", -16 * sum(xm_c[0]))
    if s_v:
        _visc_bytes(add, s_v, it_v, fused_v, merged_v, dev_v)
        if merged_v and xm_v:
            add("iso_pcg_m", -16 * sum(xm_v[0]))
    return B


def _rkl2_stage_bytes(add, kind, s, dev, c=1):
    """Stages 2..s: Fig. 2 form, or deviation form for stages 2..s-1 (the last one adds Y0 back)."""
    if dev and s >= 3:
        add(kind + "_dstage", (s - 2) * bytes_per_cell(kind + "_dstage", c))
        add(kind + "_stage", bytes_per_cell(kind + "_stage", c))
    else:
        add(kind + "_stage", (s - 1) * bytes_per_cell(kind + "_stage", c))


def _cond_bytes(add, s_c, it_c, fused, merged=False, dev=False):
    add("face_kappa", bytes_per_cell("face_kappa"))
    add("vertex_coef", bytes_per_cell("vertex_coef"))   # once per step (resident binding: RKL2 and PCG share it)
    add("aniso_gersh", bytes_per_cell("aniso_gersh"))
    add("aniso_rkl2_first", bytes_per_cell("aniso_rkl2_first"))
    _rkl2_stage_bytes(add, "aniso_rkl2", s_c, dev)
    add("aniso_pcg_r0", bytes_per_cell("aniso_pcg_r0"))
    for k in range(1, it_c + 1):
        if merged:
            add("aniso_pcg_m", bytes_per_cell("aniso_pcg_m", first=k == 1))
            continue
        if fused:
            add("aniso_pcg_s", bytes_per_cell("aniso_pcg_s", first=k == 1))
        else:
            add("pcg_pupdate", bytes_per_cell("pcg_pupdate", 1, first=k == 1))
            add("aniso_pcg_ap", bytes_per_cell("aniso_pcg_ap"))
        add("pcg_update", bytes_per_cell("pcg_update", 1))
    if it_c:
        add("pcg_xfinal", bytes_per_cell("pcg_xfinal", 1))


def _visc_bytes(add, s_v, it_v, fused=False, merged=False, dev=False):
    add("iso_gersh", bytes_per_cell("iso_gersh"))
    add("iso_rkl2_first", bytes_per_cell("iso_rkl2_first", 3))
    _rkl2_stage_bytes(add, "iso_rkl2", s_v, dev, 3)
    add("iso_pcg_r0", bytes_per_cell("iso_pcg_r0_m" if merged else "iso_pcg_r0", 3))
    if merged:   # metric-folded K1, K2, K3, wV once per binding (timed with the vertex coefficients)
        add("vertex_coef", 64)
    for k in range(1, max(it_v) + 1):
        act = sum(1 for i in it_v if i >= k)          # components still iterating at iteration k
        if merged:
            add("iso_pcg_m", bytes_per_cell("iso_pcg_m", active=act, first=k == 1))
            continue
        if fused:
            add("iso_pcg_s", bytes_per_cell("iso_pcg_s", active=act, first=k == 1))
            add("pcg_update", bytes_per_cell("pcg_update_noz", active=act))
        else:
            add("pcg_pupdate", bytes_per_cell("pcg_pupdate", active=act, first=k == 1))
            add("iso_pcg_ap", bytes_per_cell("iso_pcg_ap", active=act))
            add("pcg_update", bytes_per_cell("pcg_update", active=act))
    n_fin = sum(1 for i in it_v if i > 0)
    if n_fin:
        add("pcg_xfinal", bytes_per_cell("pcg_xfinal", active=n_fin))


# ----------------------------------------------------------------------------
# clocks during the timed region
# ----------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,utilization.gpu,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                rows.append({"sm": float(p[0]), "max": float(p[1]), "util": float(p[3]),
                             "hw": p[5], "hw_th": p[6], "sw_th": p[7], "pcap": p[8]})
            except ValueError:
                continue
        load = [r for r in rows if r["util"] >= 50] or rows
        if not load:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        reasons = set()
        for r in load:
            for key, name in (("hw", "hw_slowdown"), ("hw_th", "hw_thermal_slowdown"),
                              ("sw_th", "sw_thermal_slowdown"), ("pcap", "sw_power_cap")):
                if r[key].lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(r["sm"] for r in load), "sm_max_mhz": max(r["max"] for r in load),
                "reasons": sorted(reasons), "samples": len(load)}


# ----------------------------------------------------------------------------
# the GPU step
# ----------------------------------------------------------------------------
class Step:
    """One bench step on device-resident inputs: conduction then viscosity, through the
    resident-coefficient API (include/sts_b200.h "Resident coefficients"): the face
    diffusivities are written into the handle's binding, so the frozen vertex
    coefficients and the Gershgorin bound are built once per step and shared by the RKL2
    super-step and the PCG solve."""

    def __init__(self, G, inp, ratio, dev):
        self.G, self.inp, self.ratio = G, inp, ratio
        shape = G.shape
        alloc = lambda *s: torch.empty(s, dtype=torch.float64, device=dev)  # noqa: E731
        self.T_rk, self.T_be = alloc(*shape), alloc(*shape)
        self.v_rk, self.v_be = alloc(3, *shape), alloc(3, *shape)

    def cond(self):
        from paper_1610_01265_b200 import sts
        G, I = self.G, self.inp
        if "T" not in I:
            return 0, 0
        # conduction (anisotropic Spitzer, lagged kappa)
        T = I["T"]
        G.bind_coeffs("aniso", None, b=I["b"])
        G.face_kappa_spitzer(T, I["kappa0"], I["T_cut"], resident=True)
        dte = G.dt_euler("aniso", None)
        dt = self.ratio * dte
        s_c = sts.rkl2_num_stages(dt, dte)
        G.rkl2_advance("aniso", T, None, dt=dt, s=s_c, out=self.T_rk)
        _, (it_c,) = G.be_pcg_solve("aniso", T, None, dt=dt, rtol=RTOL, kmax=KMAX, out=self.T_be)
        self.xm_c = G.pcg_xmodes(1)
        return s_c, it_c

    def visc(self):
        from paper_1610_01265_b200 import sts
        G, I = self.G, self.inp
        if "v" not in I:
            return 0, [0]
        # viscosity (isotropic, weighted by rho, 3 components)
        v = I["v"]
        G.bind_coeffs("iso", I["visc_faces"], w=I["rho"])
        dtev = G.dt_euler("iso", None)
        dtv = self.ratio * dtev
        s_v = sts.rkl2_num_stages(dtv, dtev)
        G.rkl2_advance("iso", v, None, dt=dtv, s=s_v, out=self.v_rk)
        _, it_v = G.be_pcg_solve("iso", v, None, dt=dtv, rtol=RTOL, kmax=KMAX, out=self.v_be)
        self.xm_v = G.pcg_xmodes(3)
        return s_v, it_v

    def __call__(self):
        self.xm_c, self.xm_v = ([0], [0]), ([0, 0, 0], [0, 0, 0])
        s_c, it_c = self.cond()
        s_v, it_v = self.visc()
        return {"s_cond": s_c, "it_cond": it_c, "s_visc": s_v, "it_visc": it_v,
                "units": s_c + it_c + s_v + max(it_v), "xm_c": self.xm_c, "xm_v": self.xm_v}


class E2EStep:
    """The same step end to end through the library's HOST-ARRAY path: every input is a
    pinned host tensor passed straight to the C ABI (include/sts_b200.h "Array
    arguments"), every result lands in a pinned host tensor.  The library stages the
    arrays on its own copy streams (uploads and downloads overlap the computation of the
    calls around them), the coefficients are bound per step (uploaded into the handle's
    resident copies while the previous step still computes), and the PCG solves are
    enqueued with be_pcg_solve_async, so the host waits only where it needs a value
    (the two dt_exp, each behind the previous step's solve of the same operator only).
    The caller's stream joins the handle's copies at the end."""

    def __init__(self, G, host_inp, ratio):
        self.G, self.h, self.ratio = G, host_inp, ratio
        pin = lambda *s: torch.empty(s, dtype=torch.float64, pin_memory=True)  # noqa: E731
        shape = G.shape
        self.out = [{"T_rk": pin(*shape), "T_be": pin(*shape), "v_rk": pin(3, *shape), "v_be": pin(3, *shape)}
                    for _ in range(2)]
        nb = lambda t: t.numel() * t.element_size()  # noqa: E731
        h = host_inp
        # uploads per step: T (face kappa, RKL2, PCG), b, v (RKL2, PCG), rho, the 3 face fields
        self.h2d = 3 * nb(h["T"]) + nb(h["b"]) + 2 * nb(h["v"]) + nb(h["rho"]) + sum(nb(x) for x in h["visc_faces"])
        self.d2h = sum(nb(t) for t in self.out[0].values())
        self.n = 0

    def __call__(self):
        from paper_1610_01265_b200 import sts
        G, h, r = self.G, self.h, self.ratio
        o = self.out[self.n % 2]
        self.n += 1
        # conduction: its binding work waits for the previous step's conduction solve only
        # (the library orders it after the binding's last readers), so it overlaps the
        # previous step's viscosity
        G.bind_coeffs("aniso", None, b=h["b"])
        G.face_kappa_spitzer(h["T"], h["kappa0"], h["T_cut"], resident=True)
        dte = G.dt_euler("aniso", None)
        s_c = sts.rkl2_num_stages(r * dte, dte)
        G.rkl2_advance("aniso", h["T"], None, dt=r * dte, s=s_c, out=o["T_rk"])
        _, rc = G.be_pcg_solve_async("aniso", h["T"], None, dt=r * dte, rtol=RTOL, kmax=KMAX, out=o["T_be"])
        # viscosity: likewise behind the previous step's viscosity, while this step's
        # conduction computes
        G.bind_coeffs("iso", h["visc_faces"], w=h["rho"])
        dtev = G.dt_euler("iso", None)
        s_v = sts.rkl2_num_stages(r * dtev, dtev)
        G.rkl2_advance("iso", h["v"], None, dt=r * dtev, s=s_v, out=o["v_rk"])
        _, rv = G.be_pcg_solve_async("iso", h["v"], None, dt=r * dtev, rtol=RTOL, kmax=KMAX, out=o["v_be"])
        return {"s_cond": s_c, "s_visc": s_v, "res_c": rc, "res_v": rv}

    @staticmethod
    def units(info):
        return info["s_cond"] + info["res_c"].iters[0] + info["s_visc"] + max(info["res_v"].iters)


def dist_info():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    lrank = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, lrank


def allreduce_max(x, dev, ws):
    if ws == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws, dev):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier(device_ids=[dev.index])


# ----------------------------------------------------------------------------
# oracle CPU sample (cpu_baseline and --impl reference)
# ----------------------------------------------------------------------------
def cpu_box_config(name):
    """BASELINE config `name`'s recipe restricted to a CPU_BOX block at the
    stiff inner boundary (r planes 0.., equatorial theta band, phi 0..)."""
    _, shape, _ = W.CONFIGS[name]
    g = W.spherical_grid(*shape)
    n1, n2, n3 = CPU_BOX
    j0 = shape[1] // 2 - n2 // 2
    box = W.Grid("spherical", g.x1f[:n1 + 1], g.x2f[j0:j0 + n2 + 1], g.x3f[:n3 + 1], periodic3=False,
                 x1c=g.x1c[:n1], x2c=g.x2c[j0:j0 + n2], x3c=g.x3c[:n3], x1_span=g.span1)
    cfg = {"grid": box, **W.SPITZER}
    cfg["T"] = W.tr_corona_T(box, seed=2)
    cfg["b"] = W.multipole_b(box, seed=3)
    cfg["rho"], cfg["visc_faces"], cfg["v"] = W.viscosity_inputs(box, seed=4)
    return cfg


def oracle_step(cfg, ratio):
    from oracle import core as O
    g = cfg["grid"]
    T = cfg["T"].numpy()
    kap = O.spitzer_face_kappa(g, T, cfg["kappa0"], cfg["T_cut"])
    op = O.Operator(g, kap, cfg["b"].numpy())
    dte = O.dt_euler(op)
    dt = ratio * dte
    s_c = O.rkl2_num_stages(dt, dte)
    O.rkl2_advance(lambda x: (op.M @ x.ravel()).reshape(x.shape), T, dt, s_c)
    _, it_c = O.be_pcg_solve(op, T, dt, rtol=RTOL)
    opv = O.Operator(g, [f.numpy() for f in cfg["visc_faces"]], None, cfg["rho"].numpy())
    dtev = O.dt_euler(opv)
    s_v = O.rkl2_num_stages(ratio * dtev, dtev)
    O.rkl2_advance(opv.apply, cfg["v"].numpy(), ratio * dtev, s_v)
    _, it_v = O.be_pcg_solve(opv, cfg["v"].numpy(), ratio * dtev, rtol=RTOL)
    return s_c + it_c[0] + s_v + max(it_v)


def oracle_step_c(cfg, ratio):
    """The same step with the plain-C oracle (oracle/c/sts_oracle.c, single thread)."""
    from oracle import c_oracle as C
    g = cfg["grid"]
    T, b = cfg["T"].numpy(), cfg["b"].numpy()
    kap = C.face_kappa(g, T, cfg["kappa0"], cfg["T_cut"])
    dte = C.dt_euler(g, kap, b)
    dt = ratio * dte
    s_c = C.rkl2_num_stages(dt, dte)
    C.rkl2_advance(g, T, kap, b, None, dt, s_c)
    _, it_c = C.be_pcg_solve(g, T, kap, b, None, dt, RTOL)
    kv, rho, v = [f.numpy() for f in cfg["visc_faces"]], cfg["rho"].numpy(), cfg["v"].numpy()
    dtev = C.dt_euler(g, kv, None, rho)
    s_v = C.rkl2_num_stages(ratio * dtev, dtev)
    C.rkl2_advance(g, v, kv, None, rho, ratio * dtev, s_v)
    _, it_v = C.be_pcg_solve(g, v, kv, None, rho, ratio * dtev, RTOL)
    return s_c + it_c[0] + s_v + max(it_v)


def time_oracle(name, ratio, steps=1, warmup=0):
    """The plain-C oracle (BASELINE north_star) timed on one host core."""
    from threadpoolctl import threadpool_limits
    cfg = cpu_box_config(name)
    ncells = cfg["grid"].ncells
    from oracle import c_oracle as C
    C.set_threads(1)                 # (the C oracle's OpenMP loops: one host core, as reported)
    with threadpool_limits(limits=1):
        torch.set_num_threads(1)
        for _ in range(warmup):
            oracle_step_c(cfg, ratio)
        t0 = time.perf_counter()
        units = 0
        for _ in range(steps):
            units += oracle_step_c(cfg, ratio)
        dt = time.perf_counter() - t0
    return {"value": ncells * units / dt / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"oracle (plain C, gcc -O2, 1 thread) full step of {name}'s recipe on a "
                      f"{'x'.join(map(str, CPU_BOX))} block at r_min ({ncells} cells), dt = {ratio:g} dt_exp of "
                      f"the block, {steps} step(s): {units} cell-updates per cell in {dt:.1f} s"}, dt / steps


def run_reference(args):
    ws, rank, _ = dist_info()
    if rank != 0:
        return 0
    ratio = RATIO[args.config]
    base, sec = time_oracle(args.config, ratio, steps=args.steps, warmup=args.warmup)
    line = {"impl": "reference", "metric": METRIC, "value": base["value"], "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": args.config + " (bounded oracle sample)",
                                            "sample": base["sample"]},
            "cpu_baseline": base,
            "e2e": {"value": base["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------
def measure_device(G, inp, ratio, args, ws, dev, ncells_local, ncells_total):
    """Warm-up + the timed region on device-resident inputs, then instrumented steps for
    the per-kernel-class breakdown and the roofline of the dominant kernel."""
    step = Step(G, inp, ratio, dev)
    stream = torch.cuda.current_stream()
    for _ in range(max(args.warmup, 0)):
        step()
    launches0 = G.kernel_launches
    sampler = ClockSampler(dev.index)
    sampler.start()
    barrier(ws, dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    infos = [step() for _ in range(args.steps)]
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(ws, dev)
    clocks = sampler.stop()
    ms = allreduce_max(e0.elapsed_time(e1), dev, ws)
    launches = G.kernel_launches - launches0
    units = sum(i["units"] for i in infos)
    value = ncells_total * units / (ms * 1e-3) / 1e9

    # per-kernel-class device time: separate instrumented steps (CUDA events around every
    # launch on its stream), OUTSIDE the timed region above
    G.set_timing(True)
    G.timing_reset()
    torch.cuda.synchronize()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    pinfos = [step() for _ in range(max(1, min(args.steps, args.timing_steps)))]
    p1.record(stream)
    torch.cuda.synchronize()
    timing = G.timing()
    G.set_timing(False)
    ms_prof = p0.elapsed_time(p1)

    peak, peak_kind = peaks()
    Bytes = {}
    has = lambda k: timing.get(k, (0, 0.0))[0] > 0  # noqa: E731
    for i in pinfos:
        for k, v in algorithmic_bytes(ncells_local, i["s_cond"], i["it_cond"], i["s_visc"], i["it_visc"],
                                      has("aniso_pcg_s"), has("iso_pcg_s"), has("aniso_pcg_m"), has("iso_pcg_m"),
                                      has("aniso_rkl2_dstage"), has("iso_rkl2_dstage"), i.get("xm_c"),
                                      i.get("xm_v")).items():
            Bytes[k] = Bytes.get(k, 0.0) + v
    kernels = {}
    for k, (n, kms) in timing.items():
        if n == 0:
            continue
        ent = {"launches": n, "ms": round(kms, 3), "share": round(kms / ms_prof, 4)}
        if k in Bytes and kms > 0:
            ent["achieved_gbs"] = round(Bytes[k] / (kms * 1e-3) / 1e9, 1)
            ent["frac"] = round(ent["achieved_gbs"] / peak, 4)
        if k in KERNEL_NOTES:
            ent["note"] = KERNEL_NOTES[k]
        kernels[k] = ent
    dom = max((k for k in kernels if "achieved_gbs" in kernels[k]), key=lambda k: kernels[k]["ms"])
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        if dom in tr.get("dram_bytes_per_cell", {}) and tr.get("cells") == ncells_local:
            traffic = tr["dram_bytes_per_cell"][dom] * ncells_local
    except Exception:
        pass
    i0f = pinfos[0]
    n_eff = {"aniso_rkl2_stage": i0f["s_cond"] - 1, "aniso_pcg_ap": i0f["it_cond"],
             "aniso_pcg_s": i0f["it_cond"], "iso_rkl2_stage": i0f["s_visc"] - 1,
             "iso_pcg_ap": max(i0f["it_visc"]), "iso_pcg_s": max(i0f["it_visc"]),
             "aniso_pcg_m": i0f["it_cond"], "iso_pcg_m": max(i0f["it_visc"]),
             "aniso_rkl2_dstage": i0f["s_cond"] - 2, "iso_rkl2_dstage": i0f["s_visc"] - 2}.get(dom)
    bpl = (Bytes[dom] / len(pinfos) / n_eff) if n_eff else None
    roofline = {"bound": "hbm", "kernel": dom, "achieved": kernels[dom]["achieved_gbs"], "peak": peak,
                "unit": "GB/s", "frac": kernels[dom]["frac"], "traffic": traffic,
                "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)" if peak_kind == "measured" else "fallback",
                "algorithmic_bytes_per_launch": bpl}
    return {"value": value, "ms": ms, "infos": infos, "launches": launches, "clocks": clocks, "kernels": kernels,
            "roofline": roofline, "step": step}


def config_block(args, gg, ratio, ws, info, ncells_total, nvirt):
    return {"workload": args.config, "shape": list(gg.shape), "cells": ncells_total,
            "dt_over_dt_exp": ratio, "pcg_rtol": RTOL,
            "parallelism": f"r-slab x{ws}" + (f" (x{nvirt} virtual slabs per GPU)" if nvirt > 1 else "") +
                           (", halo exchange overlapped with interior planes" if args.halo_overlap else ""),
            "l2": f"inputs larger than L2 ({ncells_total * 8 / 1e9:.2f} GB per field)" if
            ncells_total * 8 > 126e6 else "inputs fit L2 (no flush)",
            "stages_cond": info["s_cond"], "pcg_iters_cond": info["it_cond"],
            "stages_visc": info["s_visc"], "pcg_iters_visc": info["it_visc"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4_scale512", choices=list(RATIO))
    ap.add_argument("--impl", default="sts", choices=["sts", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=-1,
                    help="end-to-end steps through the host-array path (default: as many as --steps; 0 skips)")
    ap.add_argument("--timing-steps", type=int, default=2,
                    help="instrumented steps (after the timed region) for the per-kernel breakdown")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shape", default=None, help="override n1,n2,n3 (debug)")
    ap.add_argument("--ratios", default=None,
                    help="comma-separated dt/dt_exp values: one device-timed JSON line each (e.g. the "
                         "configs[3] sweep 10,100,1000); skips the e2e and CPU legs")
    ap.add_argument("--halo-overlap", action="store_true",
                    help="decomposed grids: interior planes during the halo exchange, boundary planes after")
    ap.add_argument("--virtual", type=int, default=1,
                    help="emulate an N-way r-slab decomposition on each GPU (halo exchange through halo "
                         "buffers, the multi-GPU schedule) to measure its overhead")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    ws, rank, lrank = dist_info()
    assert ws == args.gpus or ws == 1, "launch N>1 with torchrun --nproc-per-node N"
    dev = torch.device("cuda", lrank)
    torch.cuda.set_device(dev)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    import __graft_entry__
    if rank == 0:
        __graft_entry__.build()
    barrier(ws, dev)
    from paper_1610_01265_b200 import sts

    shape = tuple(int(x) for x in args.shape.split(",")) if args.shape else None
    n1 = (shape or W.CONFIGS[args.config][1])[0]
    i0, nl = W.split_planes(n1, ws)[rank]
    cfg = W.make_config(args.config, device=dev, shape=shape, slab=(i0, nl) if ws > 1 else None)
    gg = cfg["global_grid"]
    G = sts.Grid.from_grid(gg, i0=i0, nl=nl, n_virtual=args.virtual, device=lrank)
    G.set_halo_overlap(args.halo_overlap)
    if ws > 1:
        import torch.distributed as dist
        obj = [sts.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        G.comm_init(ws, rank, obj[0])
        print(f"[bench] rank {rank}/{ws}: NCCL communicator initialised (r-slab planes [{i0}, {i0 + nl}) of {n1}, "
              f"device {lrank})", file=sys.stderr, flush=True)
    ncells_local = nl * gg.shape[1] * gg.shape[2]
    ncells_total = gg.ncells
    inp = {k: cfg[k] for k in ("T", "b", "rho", "visc_faces", "v", "kappa0", "T_cut") if k in cfg}

    if args.ratios:
        for r in [float(x) for x in args.ratios.split(",")]:
            m = measure_device(G, inp, r, args, ws, dev, ncells_local, ncells_total)
            if rank == 0:
                print(json.dumps({
                    "metric": METRIC, "value": m["value"], "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                    "warmup": args.warmup, "ms_per_step": m["ms"] / args.steps, "higher_is_better": True,
                    "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                    "config": config_block(args, gg, r, ws, m["infos"][0], ncells_total, args.virtual),
                    "roofline": m["roofline"], "gpu_launches": m["launches"], "clocks": m["clocks"],
                    "kernels": m["kernels"]}), flush=True)
            del m
        if ws > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return 0

    ratio = RATIO[args.config]
    stream = torch.cuda.current_stream()
    m = measure_device(G, inp, ratio, args, ws, dev, ncells_local, ncells_total)
    step = m.pop("step")

    # ---------------- end-to-end through the C ABI's host-array path
    e2e = None
    if args.e2e_steps < 0:
        args.e2e_steps = args.steps
    if args.e2e_steps > 0:
        del step
        torch.cuda.empty_cache()
        host_inp = dict(inp)
        for key in ("T", "b", "rho", "v"):
            host_inp[key] = inp[key].cpu().pin_memory()
        host_inp["visc_faces"] = tuple(x.cpu().pin_memory() for x in inp["visc_faces"])
        inp.clear()            # (the device inputs of the device-timed leg: the e2e leg uploads its own)
        G.unbind_coeffs("aniso")
        G.unbind_coeffs("iso")
        torch.cuda.empty_cache()
        G.async_host = True
        hstep = E2EStep(G, host_inp, ratio)
        for _ in range(3):     # warm-up (staging pool, resident copies: two steps in flight)
            hstep()
        G.join(stream)
        barrier(ws, dev)
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        hinfos = [hstep() for _ in range(args.e2e_steps)]
        G.join(stream)
        t1.record(stream)
        torch.cuda.synchronize()
        barrier(ws, dev)
        hms = allreduce_max(t0.elapsed_time(t1), dev, ws)
        assert all(i["res_c"].status == 0 and i["res_v"].status == 0 for i in hinfos)
        hunits = sum(E2EStep.units(i) for i in hinfos)
        e2e = {"value": ncells_total * hunits / (hms * 1e-3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": hstep.h2d * ws, "d2h_bytes_per_step": hstep.d2h * ws,
               "steps": args.e2e_steps, "ms_per_step": hms / args.e2e_steps,
               "mode": "C-ABI host-array path: pinned host tensors passed straight to the library calls "
                       "(face kappa, coefficient binding, dt_exp, RKL2, be_pcg_solve_async); the library stages "
                       "them on its own H2D / D2H copy streams overlapped with the computation; timed region "
                       "ends when the caller's stream has joined the last result download"}
        del host_inp, hstep

    cpu_base = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu_base, _ = time_oracle(args.config, ratio, steps=1, warmup=0)

    if rank == 0:
        line = {
            "metric": METRIC, "value": m["value"], "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": m["ms"] / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(args, gg, ratio, ws, m["infos"][0], ncells_total, args.virtual),
            "roofline": m["roofline"], "cpu_baseline": cpu_base, "e2e": e2e, "gpu_launches": m["launches"],
            "clocks": m["clocks"], "kernels": m["kernels"],
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
