"""Dev probe: one gradient evaluation + trajectories of a narrow-engine config (for ncu)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from hmcdata import make_problem
from paper_2507_14652_b200 import abi

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
ntraj = int(sys.argv[2]) if len(sys.argv) > 2 else 1
prob = make_problem(cfg)
C, k = prob.n_chains, prob.k
with abi.Context(prob) as c:
    print(abi.hmc_engine_info(c.ctx))
    T = torch.as_tensor(np.repeat(prob.frozen[prob.idx][None], C, 0), device="cuda").contiguous()
    LP = torch.empty(C, dtype=torch.float64, device="cuda")
    G = torch.empty(C, k, device="cuda")
    abi.hmc_grad(c.ctx, T, LP, G)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(ntraj):
        abi.hmc_trajectory(c.ctx, T, LP, G, prob.eps, prob.L, i)
    torch.cuda.synchronize()
    print("ms per trajectory", 1000 * (time.perf_counter() - t0) / ntraj)
