"""Dev: concurrent kernel timeline of trajectories (torch.profiler / CUPTI kernel records of the
graph's kernel nodes): per leapfrog step, the kernels in start order with start / end offsets
(us) and streams, the busy union, and the gaps on the critical path."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
from hmcdata import make_problem
from paper_2507_14652_b200 import abi
cfg = sys.argv[1]
C = int(sys.argv[2]) if len(sys.argv) > 2 else None
L = 4
prob = make_problem(cfg, n_chains=C)
C, k = prob.n_chains, prob.k
with abi.Context(prob) as c:
    T = torch.as_tensor(np.repeat(prob.frozen[prob.idx][None], C, 0).astype(np.float32), device="cuda").contiguous()
    LP = torch.empty(C, dtype=torch.float64, device="cuda"); G = torch.empty(C, k, device="cuda")
    abi.hmc_grad(c.ctx, T, LP, G)
    for it in range(3):
        abi.hmc_trajectory(c.ctx, T, LP, G, 1e-7, L, it)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        abi.hmc_trajectory(c.ctx, T, LP, G, 1e-7, L, 5)
        torch.cuda.synchronize()
    prof.export_chrome_trace("/tmp/tl.json")
ev = [e for e in json.load(open("/tmp/tl.json"))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
tot = ev[-1]["ts"] + ev[-1]["dur"] - t0
print(f"{cfg} C={C}: {len(ev)} kernels, {tot:.1f} us for L={L} (+ begin / MH)")
short = lambda n: n.replace("void ", "").replace("hmc::", "").split("(")[0][:38]
for e in ev:
    print(f"  {e['ts'] - t0:9.1f} {e['ts'] + e['dur'] - t0:9.1f} {e['dur']:7.1f}  s{e['args'].get('stream', '?'):<4} g{str(e['args'].get('grid', ''))[:14]:14s} {short(e['name'])}")
