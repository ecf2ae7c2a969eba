"""Dev: does splitting a config's chains into G independent contexts (concurrent captured graphs
on their own streams) raise throughput for latency-bound workloads?  Times S trajectories of L
steps for one C-chain context vs G contexts of C/G chains each, issued back to back."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from hmcdata import make_problem
from paper_2507_14652_b200 import abi
cfg = sys.argv[1]
C = int(sys.argv[2])
L, S = 20, 5
for G in [int(v) for v in sys.argv[3].split(",")]:
    probs = [make_problem(cfg, n_chains=C // G) for _ in range(G)]
    ctxs = [abi.Context(p) for p in probs]
    st = [torch.cuda.Stream() for _ in range(G)]
    state = []
    for p, c in zip(probs, ctxs):
        k = p.k
        T = torch.as_tensor(np.repeat(p.frozen[p.idx][None], C // G, 0).astype(np.float32), device="cuda").contiguous()
        LP = torch.empty(C // G, dtype=torch.float64, device="cuda"); Gr = torch.empty(C // G, k, device="cuda")
        abi.hmc_grad(c.ctx, T, LP, Gr)
        smp = torch.empty(C // G, S, k, device="cuda"); acc = torch.empty(C // G, S, dtype=torch.uint8, device="cuda")
        state.append((T, LP, Gr, smp, acc))
    torch.cuda.synchronize()
    def run(it):
        for g in range(G):
            T, LP, Gr, smp, acc = state[g]
            with torch.cuda.stream(st[g]):
                abi.hmc_sample(ctxs[g].ctx, T, LP, Gr, 1e-7, L, it, S, smp, acc, None, stream=torch.cuda.current_stream())
    run(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for r in range(3):
        run(100 + 10 * r)
    for g in range(G):
        torch.cuda.current_stream().wait_stream(st[g])
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (3 * S * L)
    print(f"{cfg} C={C} groups={G}: {ms*1000:7.1f} us per step of all chains, {C/ms*1000:9.0f} evals/s")
    for c in ctxs:
        c.close() if hasattr(c, "close") else abi.hmc_destroy(c.ctx)
