"""SURVEY §8(d) "Timing (oracle)": the fp64 oracle's FULL sampling runs for cfg1 (1 chain x 200
samples x L = 20 = 4,000 evaluations) and cfg2 (8 chains x 500 samples x L = 50 = 200,000
evaluations) on this host's cores, as it stands (sequential chains, NumPy/OpenBLAS threads) ->
profiles/r02_oracle_full_runs.json.  A reported baseline, not a target."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from hmcdata import make_problem  # noqa: E402
from oracle import hmc as ohmc  # noqa: E402

try:
    from threadpoolctl import threadpool_info
    threads = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
except Exception:
    threads = None
out = {"cores": len(os.sched_getaffinity(0)), "blas_threads": threads, "runs": {}}
for cfg in (sys.argv[1:] or ["cfg1", "cfg2"]):
    prob = make_problem(cfg)
    t = ohmc.Target(prob)
    th0 = prob.frozen[prob.idx].astype(np.float64)
    t0 = time.perf_counter()
    acc = []
    for ch in range(prob.n_chains):
        _, a, _ = ohmc.sample_chain(t, th0, prob.eps, prob.L, 0, prob.S, int(prob.chain_ids[ch]))
        acc.append(a.mean())
    dt = time.perf_counter() - t0
    evals = prob.n_chains * prob.S * prob.L
    out["runs"][cfg] = {"chains": prob.n_chains, "samples_per_chain": prob.S, "L": prob.L, "evals": evals,
                        "seconds": dt, "evals_per_s": evals / dt, "samples_per_s": prob.n_chains * prob.S / dt,
                        "acceptance": float(np.mean(acc))}
    print(cfg, out["runs"][cfg], flush=True)
os.makedirs("gpurun_out/r2", exist_ok=True)
json.dump(out, open("gpurun_out/r2/oracle_full_runs.json", "w"), indent=1)
