"""Where the end-to-end step's time goes: pinned H2D / D2H bandwidth alone and
concurrently, and the device step vs the host-buffer step (c4 recipe, or --shape).

  python tools/e2e_probe.py [--shape 512 512 1024]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import workloads as W  # noqa: E402


def bw(fn, nbytes, reps=3):
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return nbytes / best / 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", type=int, nargs=3, default=None)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    n = 1 << 27   # 1 GiB of FP64
    h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
    d = torch.empty(n, dtype=torch.float64, device=dev)
    d2 = torch.empty(n, dtype=torch.float64, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    print("H2D GB/s", round(bw(lambda: d.copy_(h, non_blocking=True), 8 * n), 1))
    print("D2H GB/s", round(bw(lambda: h.copy_(d, non_blocking=True), 8 * n), 1))

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    print("H2D + D2H concurrent, GB/s total", round(bw(both, 16 * n), 1))
    del h, h2, d, d2

    shape = tuple(a.shape) if a.shape else None
    cfg = W.make_config("c4_scale512", device=dev, shape=shape)
    from paper_1610_01265_b200 import sts
    G = sts.Grid.from_grid(cfg["grid"])
    inp = {k: cfg[k] for k in ("T", "b", "rho", "visc_faces", "v", "kappa0", "T_cut")}
    step = bench.Step(G, inp, 300.0, dev)
    step()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize()
    ev[0].record()
    step.cond()
    ev[1].record()
    step.visc()
    ev[2].record()
    torch.cuda.synchronize()
    print("device step ms: cond", round(ev[0].elapsed_time(ev[1]), 1), "visc", round(ev[1].elapsed_time(ev[2]), 1))
    del step
    torch.cuda.empty_cache()
    host = dict(inp)
    for key in ("T", "b", "rho", "v"):
        host[key] = inp[key].cpu().pin_memory()
    host["visc_faces"] = tuple(x.cpu().pin_memory() for x in inp["visc_faces"])
    del inp, cfg
    torch.cuda.empty_cache()
    E = bench.E2EStep(G, host, 300.0, dev)
    cs = torch.cuda.current_stream()
    E.start()
    E(prefetch=False)
    E.finish(cs)
    torch.cuda.synchronize()
    for k in (1, 3):
        E.start()
        t0 = time.perf_counter()
        for i in range(k):
            E(prefetch=i + 1 < k)
        E.finish(cs)
        torch.cuda.synchronize()
        print(f"e2e ms per step over {k} pipelined step(s) (wall)", round(1e3 * (time.perf_counter() - t0) / k, 1),
              "h2d GB", round(E.h2d / 1e9, 2), "d2h GB", round(E.d2h / 1e9, 2))


if __name__ == "__main__":
    main()
