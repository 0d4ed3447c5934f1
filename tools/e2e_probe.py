"""Per-step timeline of bench.py's end-to-end (host-array path) leg at configs[4]:
host time of every library call, device step time, the handle's memory."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import workloads as W  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    from paper_1610_01265_b200 import sts
    cfg = W.make_config("c4_scale512", device=dev)
    G = sts.Grid.from_grid(cfg["grid"])
    h = {k: cfg[k] for k in ("kappa0", "T_cut")}
    for key in ("T", "b", "rho", "v"):
        h[key] = cfg[key].cpu().pin_memory()
    h["visc_faces"] = tuple(x.cpu().pin_memory() for x in cfg["visc_faces"])
    del cfg
    torch.cuda.empty_cache()
    G.async_host = True
    st = bench.E2EStep(G, h, 300.0)
    calls = []
    orig = {}
    for name in ("bind_coeffs", "face_kappa_spitzer", "dt_euler", "rkl2_advance", "be_pcg_solve_async"):
        f = getattr(G, name)
        orig[name] = f

        def wrap(*a, _f=f, _n=name, **k):
            t = time.perf_counter()
            r = _f(*a, **k)
            calls.append((_n, time.perf_counter() - t))
            return r
        setattr(G, name, wrap)
    stream = torch.cuda.current_stream()
    for n in range(6):
        calls.clear()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t = time.perf_counter()
        info = st()
        th = time.perf_counter() - t
        G.join(stream)
        e1.record(stream)
        torch.cuda.synchronize()
        free, total = torch.cuda.mem_get_info()
        print(f"step {n}: device {e0.elapsed_time(e1):.1f} ms (isolated), host enqueue {th * 1e3:.1f} ms, "
              f"handle {G.workspace_bytes / 1e9:.1f} GB, free {free / 1e9:.1f} GB, iters "
              f"{info['res_c'].iters} {info['res_v'].iters}", flush=True)
        print("   " + ", ".join(f"{c}:{t * 1e3:.1f}" for c, t in calls), flush=True)
    # pipelined: 5 steps back to back
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for n in range(5):
        calls.clear()
        t = time.perf_counter()
        st()
        print(f"pipelined step {n}: host {1e3 * (time.perf_counter() - t):.1f} ms: " +
              ", ".join(f"{c}:{t * 1e3:.1f}" for c, t in calls), flush=True)
    G.join(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    print(f"pipelined: {e0.elapsed_time(e1) / 5:.1f} ms per step")


if __name__ == "__main__":
    main()
