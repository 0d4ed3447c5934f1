run() {
  STS_TMA_DBG=$1 timeout 60 python -c "
import torch, workloads as W, numpy as np
from paper_1610_01265_b200 import sts
g = W.spherical_grid(3, 1, 40)
G = sts.Grid.from_grid(g)
G.set_tma($2)
dev = torch.device('cuda', 0)
u = torch.rand(g.shape, dtype=torch.float64, device=dev)
k = [torch.rand(g.shape, dtype=torch.float64, device=dev) for _ in range(3)]
b = W.random_unit_b(g, seed=1).to(dev)
F = G.op_apply('aniso', u, k, b); torch.cuda.synchronize(); print('dbg $1 tma $2 ok', float(F.abs().sum()))
" 2>&1 | grep -E " ok|Error" | head -1 | sed "s/^/dbg $1 tma $2: /"
}









run 0 1
