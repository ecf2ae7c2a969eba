"""Dev probe: per-call time of hmc_sample with device vs pinned-host buffers (cfg5, L = 20)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from hmcdata import make_problem
from paper_2507_14652_b200 import abi
prob = make_problem("cfg5")
C, k, L, eps = prob.n_chains, prob.k, 20, prob.eps
with abi.Context(prob) as c:
    T = torch.as_tensor(np.repeat(prob.frozen[prob.idx][None], C, 0).astype(np.float32), device="cuda")
    LP = torch.empty(C, dtype=torch.float64, device="cuda"); G = torch.empty(C, k, device="cuda")
    abi.hmc_grad(c.ctx, T, LP, G)
    S_ = torch.empty(C, 1, k, device="cuda"); A_ = torch.empty(C, 1, dtype=torch.uint8, device="cuda"); D_ = torch.empty(C, 1, dtype=torch.float64, device="cuda")
    for i in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        abi.hmc_sample(c.ctx, T, LP, G, eps, L, i, 1, S_, A_, D_)
        torch.cuda.synchronize(); print("device", time.perf_counter() - t0, flush=True)
    hT, hLP, hG = T.cpu().pin_memory(), LP.cpu().pin_memory(), G.cpu().pin_memory()
    hS = torch.empty(C, 1, k).pin_memory(); hA = torch.empty(C, 1, dtype=torch.uint8).pin_memory(); hD = torch.empty(C, 1, dtype=torch.float64).pin_memory()
    for i in range(3):
        t0 = time.perf_counter()
        abi.hmc_sample(c.ctx, hT, hLP, hG, eps, L, 10 + i, 1, hS, hA, hD)
        print("host  ", time.perf_counter() - t0, flush=True)
    hS2 = torch.empty(C, 1, k)  # pageable
    for i in range(2):
        t0 = time.perf_counter()
        abi.hmc_sample(c.ctx, hT, hLP, hG, eps, L, 20 + i, 1, None, hA, hD)
        print("host no-samples", time.perf_counter() - t0, flush=True)
