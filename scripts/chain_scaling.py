"""Dev: time per gradient evaluation of one config at several chain counts (device-timed
trajectories, configured eps; whether a workload is latency-bound: time vs chains)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from hmcdata import make_problem
from paper_2507_14652_b200 import abi
cfg = sys.argv[1]
for C in [int(v) for v in sys.argv[2].split(",")]:
    prob = make_problem(cfg, n_chains=C)
    k, L = prob.k, 20
    with abi.Context(prob) as c:
        T = torch.as_tensor(np.repeat(prob.frozen[prob.idx][None], C, 0).astype(np.float32), device="cuda").contiguous()
        LP = torch.empty(C, dtype=torch.float64, device="cuda"); G = torch.empty(C, k, device="cuda")
        abi.hmc_grad(c.ctx, T, LP, G)
        for it in range(3):
            abi.hmc_trajectory(c.ctx, T, LP, G, 1e-7, L, it)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for it in range(5):
            abi.hmc_trajectory(c.ctx, T, LP, G, 1e-7, L, 10 + it)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5 / L
        print(f"{cfg} C={C:3d}: {ms*1000:8.1f} us per eval, {C/ms*1000:10.0f} evals/s, engine {abi.hmc_engine_info(c.ctx)}")
