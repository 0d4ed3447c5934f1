import numpy as np, torch, workloads as W
from paper_1610_01265_b200 import sts
dev = torch.device("cuda", 0)
cv = W.make_config("c2_visc64", shape=(21, 19, 70))
g = cv["grid"]
kv = [f.to(dev) for f in cv["visc_faces"]]
rho, v = cv["rho"].to(dev), cv["v"].to(dev)
for tma in (True, False):
    G1 = sts.Grid.from_grid(g); G1.set_tma(tma)
    Gv = sts.Grid.from_grid(g, n_virtual=2); Gv.set_tma(tma)
    a = G1.op_apply("iso", v, kv, None, rho); b = Gv.op_apply("iso", v, kv, None, rho)
    d = (a - b).abs()
    idx = torch.nonzero(d > 0)
    print("tma", tma, "maxdiff", float(d.max()), "rel", float(d.max() / a.abs().max()), "n", idx.shape[0], idx[:5].tolist())
G0 = sts.Grid.from_grid(g); G0.set_tma(False)
G1 = sts.Grid.from_grid(g); G1.set_tma(True)
a = G0.op_apply("iso", v, kv, None, rho); b = G1.op_apply("iso", v, kv, None, rho)
d = (a - b).abs(); idx = torch.nonzero(d > 1e-12 * a.abs().max())
print("single tma vs cp.async: rel", float(d.max() / a.abs().max()), "n", idx.shape[0], idx[:8].tolist())
