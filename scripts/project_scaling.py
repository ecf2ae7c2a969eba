"""Projection of DATA-mode strong scaling from ONE GPU (there is one GPU per call here): for
G = 1, 2, 4, 8, rank 0's shard of the G-rank job (cfg5: POINTS_XB, cfg3: ROWS) runs as a context
with hmc_config.exchange = 2 - the all-gather / reduce-scatter replaced by local copies of the same
bytes, the all-reduce skipped - so its device time is one rank's compute share.  Projected
efficiency = T(1) / (G T_rank(G)) counts compute only; the exchange (cfg5 ~68 MB
per GPU per leapfrog step at G = 8) is overlapped with the trunk except the final all-reduce.
Writes profiles/r02_scaling_projection.json.  Results of exchange = 2 contexts are not the
posterior - timing only."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from hmcdata import make_problem  # noqa: E402
from paper_2507_14652_b200 import abi  # noqa: E402
from paper_2507_14652_b200 import dist as pdist  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 3
shard = sys.argv[3] if len(sys.argv) > 3 else {"cfg5": "points_xc", "cfg3": "rows", "cfg4": "rows"}.get(cfg, "rows")
prob = make_problem(cfg)
C, k, L = prob.n_chains, prob.k, prob.L
eps = {"cfg5": 4e-7, "cfg4": 1.1e-6}.get(cfg, prob.eps)
res = {"cfg": cfg, "shard": shard, "L": L, "chains": C, "steps": K, "per_G": {}}
torch.cuda.set_device(0)
for G in (1, 2, 4, 8):
    if G == 1:
        ctx = abi.Context(prob)
    else:
        sh, n_global = {"points_xb": pdist.shard_points_xb, "points_xc": pdist.shard_points_xc,
                        "rows": pdist.shard_rows}[shard](prob, 0, G)
        ctx = abi.Context(sh, mode="data", rank=0, world=G, n_global=n_global, shard=shard, exchange="local")
    T = torch.as_tensor(np.repeat(prob.frozen[prob.idx][None], C, 0), device="cuda").contiguous()
    LP = torch.empty(C, dtype=torch.float64, device="cuda")
    Gr = torch.empty(C, k, device="cuda")
    abi.hmc_grad(ctx.ctx, T, LP, Gr)
    for w in range(2):
        abi.hmc_sample(ctx.ctx, T, LP, Gr, eps, L, w, 1, None, None, None)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    abi.hmc_sample(ctx.ctx, T, LP, Gr, eps, L, 10, K, None, None, None)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    res["per_G"][G] = {"ms_per_step_rank": ms, "engine": abi.hmc_engine_info(ctx.ctx)}
    # per-kernel-class device time of one (profiled, single-stream) leapfrog step of the rank
    abi.hmc_profile(ctx.ctx, True)
    abi.hmc_sample(ctx.ctx, T, LP, Gr, eps, L, 50, 1, None, None, None)
    torch.cuda.synchronize()
    cls = {}
    for name, pms, fl, by, step in abi.hmc_profile_read(ctx.ctx):
        if step == 0 and name != "body":
            cls[name] = cls.get(name, 0.0) + pms
    res["per_G"][G]["step0_ms_by_class"] = dict(sorted(cls.items(), key=lambda kv: -kv[1]))
    ctx.close()
t1 = res["per_G"][1]["ms_per_step_rank"]
for G, d in res["per_G"].items():
    d["projected_evals_per_s"] = C * L / (d["ms_per_step_rank"] / 1000.0)
    d["projected_efficiency_compute_only"] = t1 / (G * d["ms_per_step_rank"])
print(json.dumps(res, indent=1))
os.makedirs("gpurun_out/r2", exist_ok=True)
json.dump(res, open(f"gpurun_out/r2/scaling_projection_{cfg}_{shard}.json", "w"), indent=1)
