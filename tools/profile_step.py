"""Run `steps` bench steps of a config once (for ncu / compute-sanitizer captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3_spitzer256")
    ap.add_argument("--visc", action="store_true", help="add the c4 viscosity inputs")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--twopass", action="store_true", help="two-pass S / U PCG iteration instead of merged")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    from paper_1610_01265_b200 import sts
    name = "c4_scale512" if a.visc else a.config
    shape = W.CONFIGS[a.config][1]
    cfg = W.make_config(name, device=dev, shape=shape)
    G = sts.Grid.from_grid(cfg["grid"])
    G.set_pcg_merged(not a.twopass)
    inp = {k: cfg[k] for k in ("T", "b", "rho", "visc_faces", "v", "kappa0", "T_cut") if k in cfg}
    step = bench.Step(G, inp, 300.0, dev)
    for _ in range(a.steps):
        print(step(), flush=True)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
