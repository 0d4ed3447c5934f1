"""Two ranks through the library over NCCL (one process per GPU, r-slab per rank):
operator and RKL2 bit-identical to the single domain, PCG to rounding.  Needs >= 2
visible GPUs (skipped otherwise; the round's GPU boxes have one -- the host-side logic
of the decomposition is covered by tests/test_dist_gloo.py on CPU)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r'''
import os, sys
sys.path.insert(0, os.environ["STS_ROOT"])
import numpy as np, torch, torch.distributed as dist
import workloads as W
from paper_1610_01265_b200 import sts
rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = torch.device("cuda", rank)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
cfg = W.make_config("c1_spitzer64", shape=(24, 19, 64), device=dev)
g = cfg["grid"]
i0, nl = W.split_planes(g.shape[0], ws)[rank]
G = sts.Grid.from_grid(g, i0=i0, nl=nl, device=rank)
obj = [sts.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
G.comm_init(ws, rank, obj[0])
sl = slice(i0, i0 + nl)
T, b = cfg["T"][sl].contiguous(), cfg["b"][:, sl].contiguous()
k = G.face_kappa_spitzer(T, cfg["kappa0"], cfg["T_cut"])
dte = G.dt_euler("aniso", k, b)
s = sts.rkl2_num_stages(100 * dte, dte)
F = G.op_apply("aniso", T, k, b)
u = G.rkl2_advance("aniso", T, k, b, None, 100 * dte, s)
x, it = G.be_pcg_solve("aniso", T, k, b, None, 100 * dte, 1e-12, 10000)
outs = [torch.zeros_like(cfg["T"]) for _ in range(3)]
for o, part in zip(outs, (F, u, x)):
    full = [torch.zeros((n,) + tuple(g.shape[1:]), dtype=torch.float64, device=dev)
            for _, n in W.split_planes(g.shape[0], ws)]
    dist.all_gather(full, part)
    o.copy_(torch.cat(full))
if rank == 0:
    G1 = sts.Grid.from_grid(g, device=0)
    k1 = G1.face_kappa_spitzer(cfg["T"], cfg["kappa0"], cfg["T_cut"])
    assert G1.dt_euler("aniso", k1, cfg["b"]) == dte
    assert torch.equal(outs[0], G1.op_apply("aniso", cfg["T"], k1, cfg["b"]))
    assert torch.equal(outs[1], G1.rkl2_advance("aniso", cfg["T"], k1, cfg["b"], None, 100 * dte, s))
    x1, i1 = G1.be_pcg_solve("aniso", cfg["T"], k1, cfg["b"], None, 100 * dte, 1e-12, 10000)
    assert abs(i1[0] - it[0]) <= 1
    assert float((outs[2] - x1).norm() / x1.norm()) <= 1e-12
    print("NCCL 2-rank OK", it, i1)
dist.destroy_process_group()
'''


def test_two_ranks_over_nccl_match_single_domain(tmp_path):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    import __graft_entry__ as e
    e.build()
    w = tmp_path / "worker.py"
    w.write_text(WORKER)
    env = dict(os.environ, STS_ROOT=ROOT)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", "29531", str(w)],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "NCCL 2-rank OK" in r.stdout
