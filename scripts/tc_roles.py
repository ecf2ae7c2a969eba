"""Dev diagnostic: per-role barrier wait fractions of each tcgen05 GEMM variant over one cfg5
trajectory (HMC_TC_PROF=1)."""
import os, sys
os.environ["HMC_TC_PROF"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from hmcdata import make_problem
from paper_2507_14652_b200 import abi
NAMES = ["fwd", "dgrad", "wgrad", "combine", "dB", "dT", "st0", "st1", "st2", "st3"]
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
prob = make_problem(cfg)
C, k = prob.n_chains, prob.k
with abi.Context(prob) as c:
    T = torch.as_tensor(np.repeat(prob.frozen[prob.idx][None], C, 0).astype(np.float32), device="cuda")
    LP = torch.empty(C, dtype=torch.float64, device="cuda"); G = torch.empty(C, k, device="cuda")
    abi.hmc_grad(c.ctx, T, LP, G)
    abi.hmc_trajectory(c.ctx, T, LP, G, prob.eps, 4, 0)
    torch.cuda.synchronize()
    abi.hmc_debug_tc_profile(reset=True)
    abi.hmc_trajectory(c.ctx, T, LP, G, prob.eps, 10, 1)
    torch.cuda.synchronize()
    prof = abi.hmc_debug_tc_profile()
for vid, d in sorted(prof.items()):
    tot = d["kernel_cycles"] or 1
    print(f"{NAMES[vid]:8s} kernel {tot / 148 / 1e3:9.1f} kclk/CTA  " +
          "  ".join(f"{k}={100.0 * v / tot:5.1f}%" for k, v in d.items() if k != "kernel_cycles"))
