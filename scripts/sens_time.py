import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from hmcdata import make_problem
from paper_2507_14652_b200 import abi
from oracle import sensitivity as osens
for cfg in ["cfg2", "cfg3", "cfg4", "cfg5"]:
    prob = make_problem(cfg, n_chains=1)
    abi.hmc_sensitivity(prob)
    t0 = time.perf_counter(); s2 = abi.hmc_sensitivity(prob); dt = time.perf_counter() - t0
    n90 = osens.n_hat(s2, 0.9)
    print(f"{cfg}: P={s2.size} sensitivity {dt*1e3:.1f} ms (incl. context setup); N^(tau=0.9)={n90} "
          f"({100.0*n90/s2.size:.1f}%), N^(0.99)={osens.n_hat(s2, 0.99)}", flush=True)
