"""Small end-to-end run of every hot kernel for compute-sanitizer (memcheck / racecheck / synccheck).

  compute-sanitizer --tool memcheck python tools/probe/sanitize_small.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1610_01265_b200 import sts  # noqa: E402

dev = torch.device("cuda", 0)
for nv in (1, 2):
    cfg = W.make_config("c4_scale512", device=dev, shape=(12, 30, 64))
    G = sts.Grid.from_grid(cfg["grid"], n_virtual=nv)
    T, b = cfg["T"], cfg["b"]
    k = G.face_kappa_spitzer(T, cfg["kappa0"], cfg["T_cut"])
    dte = G.dt_euler("aniso", k, b)
    s = sts.rkl2_num_stages(50 * dte, dte)
    u = G.rkl2_advance("aniso", T, k, b, None, 50 * dte, s)
    x, it = G.be_pcg_solve("aniso", T, k, b, None, 50 * dte, 1e-10, 2000)
    kv, rho, v = cfg["visc_faces"], cfg["rho"], cfg["v"]
    dtv = G.dt_euler("iso", kv, None, rho)
    sv = sts.rkl2_num_stages(100 * dtv, dtv)
    uv = G.rkl2_advance("iso", v, kv, None, rho, 100 * dtv, sv)
    xv, itv = G.be_pcg_solve("iso", v, kv, None, rho, 100 * dtv, 1e-10, 2000)
    torch.cuda.synchronize()
    print("nv", nv, "stages", s, sv, "iters", it, itv, float(u.sum()), float(xv.sum()), flush=True)
