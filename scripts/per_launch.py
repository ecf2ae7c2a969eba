"""Dev: per-launch times of one profiled (single-stream) leapfrog step on cfg5."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from hmcdata import make_problem
from paper_2507_14652_b200 import abi
prob = make_problem(sys.argv[1] if len(sys.argv) > 1 else "cfg5")
C, k = prob.n_chains, prob.k
with abi.Context(prob) as c:
    T = torch.as_tensor(np.repeat(prob.frozen[prob.idx][None], C, 0).astype(np.float32), device="cuda")
    LP = torch.empty(C, dtype=torch.float64, device="cuda"); G = torch.empty(C, k, device="cuda")
    abi.hmc_grad(c.ctx, T, LP, G)
    S_ = torch.empty(C, 1, k, device="cuda"); A_ = torch.empty(C, 1, dtype=torch.uint8, device="cuda"); D_ = torch.empty(C, 1, dtype=torch.float64, device="cuda")
    abi.hmc_sample(c.ctx, T, LP, G, prob.eps, 4, 0, 1, S_, A_, D_)
    abi.hmc_profile(c.ctx, True)
    abi.hmc_sample(c.ctx, T, LP, G, prob.eps, 4, 1, 1, S_, A_, D_)
    torch.cuda.synchronize()
    for name, ms, fl, by, step in abi.hmc_profile_read(c.ctx):
        if step == 0:
            print(f"{name:14s} {ms*1000:8.1f} us {fl/ms/1e9 if ms > 0 else 0:8.1f} TF/s")
