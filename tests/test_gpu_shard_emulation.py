"""DATA mode with G = 2, 4, 8 ranks emulated on ONE GPU (SURVEY §8(c) multi-GPU parity protocol;
§8(e)).  Each rank is its own libhmc context over its shard (set up with exchange = "emulated",
i.e. no communicator); the contexts run one after another through hmc_debug_data_phase, and the
test performs each collective between the phases with plain tensor sums and concatenations:

  POINTS_XB:  phase 0 (forward)  -> all-gather of the branch outputs
              phase 1 (combine, partial dB) -> reduce-scatter of dB
              phase 2 (dT, backward) -> all-reduce of [g_lik, sum r^2]
              phase 3 (prior, log pi)
  ROWS:       phase 0 (local evaluation) -> all-reduce -> phase 3

so the library's own multi-rank code - shard validation, the k_xb_gather / k_xb_scatter
permutations for G > 1, the per-rank partial sums and the prior added once after the reduction -
runs exactly as with NCCL, and the result must match the oracle's FULL-batch gradient."""
import numpy as np
import pytest

from hmcdata import ArchSpec, NetSpec, make_problem, make_tiny_problem
from oracle import hmc as ohmc

from gpu_util import assert_grad_close, jittered_states, to_dev, torch_cuda

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("G", [2, 4, 8])
def test_xb_permutations_match_numpy(G):
    """k_xb_gather: [rank][chain][i][k] -> [chain][rank n_loc + i][k]; k_xb_scatter: its inverse."""
    torch = torch_cuda()
    from paper_2507_14652_b200 import abi
    C, n_loc, p = 3, 5, 7
    g = np.random.default_rng(G)
    recv = g.normal(size=(G, C, n_loc, p)).astype(np.float32)
    full = torch.empty(C, G * n_loc, p, device="cuda")
    abi.hmc_debug_xb_permute(0, C, G, n_loc, p, to_dev(recv, torch.float32), full)
    np.testing.assert_array_equal(full.cpu().numpy(), recv.transpose(1, 0, 2, 3).reshape(C, G * n_loc, p))
    src = g.normal(size=(C, G * n_loc, p)).astype(np.float32)
    send = torch.empty(G, C, n_loc, p, device="cuda")
    abi.hmc_debug_xb_permute(1, C, G, n_loc, p, to_dev(src, torch.float32), send)
    np.testing.assert_array_equal(send.cpu().numpy(), src.reshape(C, G, n_loc, p).transpose(1, 0, 2, 3))


def _rank_contexts(prob, G, shard):
    from paper_2507_14652_b200 import abi
    from paper_2507_14652_b200 import dist as pdist
    ctxs = []
    for r in range(G):
        sh, n_global = {"points_xb": pdist.shard_points_xb, "points_xc": pdist.shard_points_xc,
                        "rows": pdist.shard_rows}[shard](prob, r, G)
        ctxs.append(abi.Context(sh, mode="data", rank=r, world=G, n_global=n_global, shard=shard,
                                exchange="emulated"))
    return ctxs


def _emulated_grad(prob, th, G, shard):
    """log pi and gradient of every chain, as every rank would return them; checks that all
    ranks agree bitwise (they all finish from the same all-reduced sums)."""
    torch = torch_cuda()
    from paper_2507_14652_b200 import abi
    C, k = th.shape
    T = to_dev(th, torch.float32)
    ctxs = _rank_contexts(prob, G, shard)
    try:
        gl = [torch.empty(C, k, device="cuda") for _ in range(G)]
        lik = [torch.empty(C, dtype=torch.float64, device="cuda") for _ in range(G)]
        if shard == "points_xc":   # chain blocks: rank r's branch outputs are chains [r C/G, (r+1) C/G)
            n_c = prob.v.shape[0]
            p = prob.arch.nets[0].widths[-1]
            Cb = C // G
            B = [torch.empty(Cb, n_c, p, device="cuda") for _ in range(G)]
            for r, c in enumerate(ctxs):
                abi.hmc_debug_data_phase(c.ctx, 0, T, None, B[r])
            gathered = torch.cat(B).contiguous()                      # all-gather, rank (= chain) order
            send = [torch.empty(C, n_c, p, device="cuda") for _ in range(G)]
            for r, c in enumerate(ctxs):
                abi.hmc_debug_data_phase(c.ctx, 1, gathered, None, send[r])
            tot = send[0].clone()
            for q in range(1, G):
                tot += send[q]
            for r, c in enumerate(ctxs):                              # reduce-scatter: chain block r to rank r
                abi.hmc_debug_data_phase(c.ctx, 2, tot[r * Cb:(r + 1) * Cb].contiguous(), None, gl[r], lik[r])
        elif shard == "points_xb":
            n_c = prob.v.shape[0]
            p = prob.arch.nets[0].widths[-1]
            B = [torch.empty(C, n_c // G, p, device="cuda") for _ in range(G)]
            for r, c in enumerate(ctxs):
                abi.hmc_debug_data_phase(c.ctx, 0, T, None, B[r])
            gathered = torch.stack(B).contiguous()                    # all-gather, rank order
            send = [torch.empty(G, C, n_c // G, p, device="cuda") for _ in range(G)]
            for r, c in enumerate(ctxs):
                abi.hmc_debug_data_phase(c.ctx, 1, gathered, None, send[r])
            for r, c in enumerate(ctxs):                              # reduce-scatter: block r to rank r
                dB = send[0][r].clone()
                for q in range(1, G):
                    dB += send[q][r]
                abi.hmc_debug_data_phase(c.ctx, 2, dB.contiguous(), None, gl[r], lik[r])
        else:
            for r, c in enumerate(ctxs):
                abi.hmc_debug_data_phase(c.ctx, 0, T, None, gl[r], lik[r])
        gsum, lsum = gl[0].clone(), lik[0].clone()                    # all-reduce, rank order
        for r in range(1, G):
            gsum += gl[r]
            lsum += lik[r]
        outs = []
        for c in ctxs:
            g = torch.empty(C, k, device="cuda")
            lp = torch.empty(C, dtype=torch.float64, device="cuda")
            abi.hmc_debug_data_phase(c.ctx, 3, gsum.contiguous(), lsum.contiguous(), g, lp)
            outs.append((lp.cpu().numpy(), g.cpu().numpy()))
        for lp, g in outs[1:]:
            np.testing.assert_array_equal(lp, outs[0][0])
            np.testing.assert_array_equal(g, outs[0][1])
        return outs[0]
    finally:
        for c in ctxs:
            c.close()


XB_ARCH = ArchSpec("deeponet", (NetSpec.plain((7, 130, 64, 50)), NetSpec.plain((3, 70, 50), last="tanh")), has_b0=True)


@pytest.mark.parametrize("G", [2, 4, 8])
def test_points_xb_emulated_ranks_match_oracle(G):
    prob = make_tiny_problem(XB_ARCH, n_c=64, n_x=200, active_frac=0.5, n_chains=3, seed=61, noise=0.3)
    th = jittered_states(prob, 3)
    lp, g = _emulated_grad(prob, th, G, "points_xb")
    t = ohmc.Target(prob)
    for ci in range(3):
        lr, gr = t.logp_grad(th[ci])
        assert_grad_close(lp[ci], g[ci], lr, gr, f"points_xb G={G} chain {ci}")


def test_points_xb_emulated_cfg5_G8():
    """cfg5 at full size over 8 emulated ranks (each: 64 conditions x 256 points), 2 chains: the
    multi-GPU parity row of SURVEY §8(c) for the north-star config."""
    prob = make_problem("cfg5", n_chains=2)
    th = jittered_states(prob, 2)
    lp, g = _emulated_grad(prob, th, 8, "points_xb")
    t = ohmc.Target(prob)
    for ci in range(2):
        lr, gr = t.logp_grad(th[ci])
        assert_grad_close(lp[ci], g[ci], lr, gr, f"cfg5 points_xb G=8 chain {ci}")


@pytest.mark.parametrize("G", [2, 4, 8])
def test_rows_emulated_ranks_match_oracle(G):
    """Row layout: an MLP with tensor-core widths (cfg3's shape at 2,048 rows) and a DeepONet
    (function blocks, trunk replicated)."""
    mlp = make_tiny_problem(ArchSpec("mlp", (NetSpec.plain((8, 256, 256, 1)),)), n=2048, active_frac=0.05,
                            n_chains=2, seed=62, noise=0.3)
    don = make_tiny_problem(XB_ARCH, n_c=64, n_x=40, active_frac=0.5, n_chains=2, seed=63, noise=0.3)
    for prob in (mlp, don):
        th = jittered_states(prob, 2)
        lp, g = _emulated_grad(prob, th, G, "rows")
        t = ohmc.Target(prob)
        for ci in range(2):
            lr, gr = t.logp_grad(th[ci])
            assert_grad_close(lp[ci], g[ci], lr, gr, f"rows G={G} {prob.arch.kind} chain {ci}")


def test_emulated_context_refuses_the_graph_calls():
    torch = torch_cuda()
    from paper_2507_14652_b200 import abi
    prob = make_tiny_problem(XB_ARCH, n_c=16, n_x=24, n_chains=1, seed=64)
    ctxs = _rank_contexts(prob, 2, "points_xb")
    try:
        th = jittered_states(prob, 1)
        with pytest.raises(abi.HmcError) as e:
            abi.hmc_grad(ctxs[0].ctx, to_dev(th, torch.float32), torch.empty(1, dtype=torch.float64, device="cuda"),
                         torch.empty(1, prob.k, device="cuda"))
        assert e.value.code == abi.HMC_E_STATE
    finally:
        for c in ctxs:
            c.close()


@pytest.mark.parametrize("G", [2, 4, 8])
def test_points_xc_emulated_ranks_match_oracle(G):
    """POINTS_XC: the branch for this rank's chain block on all conditions, the trunk
    and the combine on its point block; 8 chains so every rank owns at least one."""
    prob = make_tiny_problem(XB_ARCH, n_c=40, n_x=200, active_frac=0.5, n_chains=8, seed=65, noise=0.3)
    th = jittered_states(prob, 8)
    lp, g = _emulated_grad(prob, th, G, "points_xc")
    t = ohmc.Target(prob)
    for ci in (0, 3, 7):
        lr, gr = t.logp_grad(th[ci])
        assert_grad_close(lp[ci], g[ci], lr, gr, f"points_xc G={G} chain {ci}")


def test_points_xc_emulated_cfg5_G8():
    """cfg5 at full size over 8 emulated ranks in the POINTS_XC layout (8 chains: one per rank)."""
    prob = make_problem("cfg5", n_chains=8)
    th = jittered_states(prob, 8)
    lp, g = _emulated_grad(prob, th, 8, "points_xc")
    t = ohmc.Target(prob)
    for ci in (0, 5):
        lr, gr = t.logp_grad(th[ci])
        assert_grad_close(lp[ci], g[ci], lr, gr, f"cfg5 points_xc G=8 chain {ci}")
