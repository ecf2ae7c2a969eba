import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from hmcdata import make_problem
from paper_2507_14652_b200 import abi
cfg = sys.argv[1]
prob = make_problem(cfg, n_chains=2)
with abi.Context(prob) as c:
    T = torch.as_tensor(np.repeat(prob.frozen[prob.idx][None], 2, 0).astype(np.float32), device="cuda")
    LP = torch.empty(2, dtype=torch.float64, device="cuda"); G = torch.empty(2, prob.k, device="cuda")
    abi.hmc_grad(c.ctx, T, LP, G)
    torch.cuda.synchronize()
    print(cfg, "grad ok", LP.cpu().numpy(), flush=True)
