"""NEXT-3 harness (§4.2.3 / Table 3): the method's gain on B200 with the
same kernels.  For a config, reduced-space HMC (k from the config's VI-sigma mask) vs full HMC
(k = P, every parameter sampled): (1) time per trajectory at the config's L (the cost of a
step is unchanged by the reduction - this measures it), (2) the dual-averaged step size for an
80 % acceptance target from the same start, (3) trajectories of length pi/2 / eps needed
per unit integration time, i.e. relative cost per sample at equal acceptance.
Usage: python scripts/cost_compare.py cfg4 [n_adapt]  -> one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from hmcdata import make_problem
from paper_2507_14652_b200 import abi

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
n_adapt = int(sys.argv[2]) if len(sys.argv) > 2 else 150
L_adapt = 20
out = {"config": cfg, "n_adapt": n_adapt, "L_adapt": L_adapt, "delta": 0.8}
for mode in ("reduced", "full"):
    prob = make_problem(cfg)
    if mode == "full":
        prob.idx = np.arange(prob.frozen.shape[0], dtype=np.int32)
    C, k = prob.n_chains, prob.idx.shape[0]
    with abi.Context(prob) as c:
        th = torch.as_tensor(np.repeat(prob.frozen[prob.idx][None], C, 0).astype(np.float32), device="cuda")
        lp = torch.empty(C, dtype=torch.float64, device="cuda")
        g = torch.empty(C, k, device="cuda")
        abi.hmc_grad(c.ctx, th, lp, g)
        # (1) time per trajectory at the config's L (after a warm-up replay)
        abi.hmc_trajectory(c.ctx, th, lp, g, prob.eps, prob.L, 0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in range(3):
            abi.hmc_trajectory(c.ctx, th, lp, g, prob.eps, prob.L, 1 + s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        # (2) adapted step for 80 % acceptance from the seeded start
        th2 = torch.as_tensor(np.repeat(prob.frozen[prob.idx][None], C, 0).astype(np.float32), device="cuda")
        abi.hmc_grad(c.ctx, th2, lp, g)
        t0 = time.perf_counter()
        eb = abi.hmc_adapt(c.ctx, th2, lp, g, prob.eps, L_adapt, 100, n_adapt, 0.8)
        t_ad = time.perf_counter() - t0
    out[mode] = {"k": int(k), "ms_per_trajectory": ms, "L": prob.L, "ms_per_gradient_eval_all_chains": ms / prob.L,
                 "eps_bar_median": float(np.median(eb)), "eps_bar_min": float(eb.min()), "eps_bar_max": float(eb.max()),
                 "adapt_seconds": t_ad}
    print(f"[{mode}] k={k} {ms:.1f} ms/trajectory (L={prob.L}), eps_bar median {np.median(eb):.3e}", file=sys.stderr)
r, f = out["reduced"], out["full"]
out["step_ratio_reduced_over_full"] = r["eps_bar_median"] / f["eps_bar_median"]
out["cost_per_eval_ratio_full_over_reduced"] = f["ms_per_gradient_eval_all_chains"] / r["ms_per_gradient_eval_all_chains"]
out["cost_per_unit_time_ratio_full_over_reduced"] = out["cost_per_eval_ratio_full_over_reduced"] * out["step_ratio_reduced_over_full"]
print(json.dumps(out))
