"""Dev diagnostic (not a test): per-layer gradient error of each GEMM engine vs the oracle."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from hmcdata import make_problem
from hmcdata.generate import layout_entries
from oracle import hmc as ohmc
from gpu_util import gpu_grad, jittered_states
from paper_2507_14652_b200 import abi

cfgs = sys.argv[1:] or ["cfg2", "cfg3", "cfg4", "cfg5"]
for cfg in cfgs:
    prob = make_problem(cfg, n_chains=2)
    th = jittered_states(prob, 2)
    t = ohmc.Target(prob)
    lr, gr = t.logp_grad(th[1])
    ent = layout_entries(prob.arch)
    for eng in ["simt", "tc"]:
        abi.hmc_debug_set_engine(1 if eng == "simt" else 0)
        with abi.Context(prob) as c:
            info = abi.hmc_engine_info(c.ctx)
            lp, g = gpu_grad(c, th)
        g1 = g[1].astype(np.float64)
        print(f"{cfg} {eng} [{info}] logp rel {abs(lp[1]-lr)/abs(lr):.3e}  grad l2 rel {np.linalg.norm(g1-gr)/np.linalg.norm(gr):.3e}", flush=True)
        for kind, off, size, fi in ent:
            sel = (prob.idx >= off) & (prob.idx < off + size)
            if sel.sum() == 0: continue
            d = np.linalg.norm(g1[sel] - gr[sel]); n = np.linalg.norm(gr[sel])
            print(f"    {kind} off={off} size={size} nact={sel.sum()} |g|={n:.3e} rel={d/max(n,1e-300):.3e}", flush=True)
