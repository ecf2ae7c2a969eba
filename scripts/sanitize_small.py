"""Dev check: one gradient evaluation of small problems of every layout (run under
compute-sanitizer)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from hmcdata import ArchSpec, NetSpec, make_tiny_problem
from gpu_util import gpu_grad, jittered_states
from paper_2507_14652_b200 import abi
D = ArchSpec("deeponet", (NetSpec.plain((7, 130, 64, 50)), NetSpec.plain((3, 70, 50), last="tanh")), has_b0=True)
M = ArchSpec("mlp", (NetSpec.plain((3, 150, 70, 1)),))
cases = [("mlp", M, dict(n=333)), ("deeponet", D, dict(n_c=40, n_x=37)),
         ("unaligned", D, dict(n_c=12, n_x=9, unaligned=True))]
for name, arch, kw in cases:
    prob = make_tiny_problem(arch, n_chains=2, seed=3, active_frac=0.5, **kw)
    th = jittered_states(prob, 2)
    with abi.Context(prob) as c:
        lp, g = gpu_grad(c, th)
    print(name, "ok", lp, flush=True)
prob = make_tiny_problem(D, n_chains=2, seed=4, active_frac=0.5, n_c=40, n_x=37)
with abi.Context(prob, mode="data", shard="points_xb") as c:
    lp, g = gpu_grad(c, jittered_states(prob, 2))
print("points_xb ok", lp, flush=True)
