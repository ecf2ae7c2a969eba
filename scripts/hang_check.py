import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from hmcdata import make_problem
from paper_2507_14652_b200 import abi
cfg = sys.argv[1]
C = int(sys.argv[2]) if len(sys.argv) > 2 else 2
prob = make_problem(cfg, n_chains=C)
with abi.Context(prob) as c:
    T = torch.as_tensor(np.repeat(prob.frozen[prob.idx][None], C, 0).astype(np.float32), device="cuda")
    LP = torch.empty(C, dtype=torch.float64, device="cuda"); G = torch.empty(C, prob.k, device="cuda")
    abi.hmc_grad(c.ctx, T, LP, G)
    torch.cuda.synchronize()
    print(cfg, C, "grad ok", LP.cpu().numpy()[:2], flush=True)
