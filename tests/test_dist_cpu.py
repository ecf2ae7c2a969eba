"""World-size-2 gloo tests (CPU) of the data-parallel host logic: row sharding, NCCL-id
broadcast, and the reduction algebra libhmc relies on in DATA mode (sum of per-shard likelihood
gradients, prior added once after the all-reduce == full-batch gradient)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from hmcdata import ArchSpec, NetSpec, make_tiny_problem
from paper_2507_14652_b200 import dist as pdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(kind):
    if kind == "mlp":
        arch = ArchSpec("mlp", (NetSpec.plain((2, 7, 5, 1)),))
        return arch, make_tiny_problem(arch, n=37, active_frac=0.5, seed=3, noise=0.4), 37
    arch = ArchSpec("deeponet", (NetSpec.plain((3, 6, 4)), NetSpec.plain((2, 5, 4), last="tanh")), has_b0=True)
    # deeponet_unaligned: per-function query points, sharded with their functions
    return arch, make_tiny_problem(arch, n_c=11, n_x=9, active_frac=0.6, seed=4, noise=0.4,
                                   unaligned=(kind == "deeponet_unaligned")), 99


def _worker(rank, world, port, kind, q):
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import hmc as ohmc
    from oracle import network as onet
    arch, prob, _ = _case(kind)
    shard, n_global = pdist.shard_rows(prob, rank, world)
    th = prob.frozen[prob.idx].astype(np.float64) + 0.01
    t = ohmc.Target(shard)
    full = t.assemble(th)
    ll, g_full, _ = onet.loglik_grad(arch, full, t.data, t.sigma)
    buf = torch.tensor(np.concatenate([g_full[prob.idx], [ll]]), dtype=torch.float64)
    dist.all_reduce(buf)                      # the DATA-mode reduction: likelihood sums only
    sp2 = prob.prior_sigma ** 2
    g = buf[:-1].numpy() - th / sp2           # prior added once, after the reduction
    lp = buf[-1].item() - np.dot(th, th) / (2 * sp2)
    # NCCL id broadcast path (any 128-byte payload)
    nid = pdist.broadcast_nccl_id(lambda: bytes(range(128)))
    q.put((rank, lp, g, n_global, nid))
    dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["mlp", "deeponet", "deeponet_unaligned"])
def test_data_mode_reduction_matches_full_batch(kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    from oracle import hmc as ohmc
    arch, prob, N = _case(kind)
    th = prob.frozen[prob.idx].astype(np.float64) + 0.01
    lp_ref, g_ref = ohmc.Target(prob).logp_grad(th)
    for rank, lp, g, n_global, nid in res:
        assert n_global == N
        assert nid == bytes(range(128))
        assert lp == pytest.approx(lp_ref, rel=1e-12)
        np.testing.assert_allclose(g, g_ref, rtol=1e-11, atol=1e-11)
    # both ranks hold bitwise-identical reduced values (MH decisions agree without a broadcast)
    np.testing.assert_array_equal(res[0][2], res[1][2])


def test_row_blocks_partition_rows():
    for n in (1, 7, 37, 1024):
        for w in (1, 2, 3, 8):
            blocks = [pdist.row_block(n, r, w) for r in range(w)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1


def test_chain_ids_are_global_and_disjoint():
    ids = [set(pdist.chain_ids(r, 64).tolist()) for r in range(8)]
    assert set.union(*ids) == set(range(512))
    assert sum(len(s) for s in ids) == 512


def _xb_worker(rank, world, port, q):
    """POINTS_XB algebra with the oracle's per-net passes: branch on this rank's conditions, trunk
    on its points, all-gather B, residual for all conditions x its points, reduce-scatter dB,
    local dT, all-reduce of the likelihood gradient and sum r^2 == the full-batch values."""
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import network as onet
    arch, prob = _xb_case()
    sh, n_global = pdist.shard_points_xb(prob, rank, world)
    th = prob.frozen.astype(np.float64) + 0.01
    B, tb = onet.net_forward(arch, th, 0, sh.u.astype(np.float64))
    T, tt = onet.net_forward(arch, th, 1, sh.q.astype(np.float64))
    parts = [torch.zeros_like(torch.as_tensor(B)) for _ in range(world)]
    dist.all_gather(parts, torch.as_tensor(B))
    Ball = torch.cat(parts).numpy()
    _, b0, _ = onet.layer_table(arch)
    s2 = prob.noise_sigma ** 2
    R = sh.v.astype(np.float64) - (Ball @ T.T + th[b0])
    E = R / s2
    g = np.zeros_like(th)
    dB_part = torch.as_tensor(E @ T)                        # all conditions, this rank's points
    dB_own = torch.zeros_like(torch.as_tensor(B))
    dist.reduce_scatter(dB_own, list(dB_part.chunk(world)))
    onet.net_backward(arch, th, 0, tb, dB_own.numpy(), g)   # branch: own conditions
    onet.net_backward(arch, th, 1, tt, E.T @ Ball, g)       # trunk: own points, all conditions
    g[b0] += E.sum()
    buf = torch.tensor(np.concatenate([g, [-np.sum(R * R) / (2 * s2)]]), dtype=torch.float64)
    dist.all_reduce(buf)
    q.put((rank, buf.numpy(), n_global))
    dist.destroy_process_group()


def _xb_case():
    arch = ArchSpec("deeponet", (NetSpec.plain((3, 6, 4)), NetSpec.plain((2, 5, 4), last="tanh")), has_b0=True)
    return arch, make_tiny_problem(arch, n_c=12, n_x=9, active_frac=0.6, seed=6, noise=0.4)


def test_points_xb_exchange_matches_full_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_xb_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import network as onet
    arch, prob = _xb_case()
    th = prob.frozen.astype(np.float64) + 0.01
    data = {"u": prob.u.astype(np.float64), "q": prob.q.astype(np.float64), "v": prob.v.astype(np.float64)}
    ll, g_ref, _ = onet.loglik_grad(arch, th, data, prob.noise_sigma)
    for rank, buf, n_global in res:
        assert n_global == 12 * 9
        np.testing.assert_allclose(buf[:-1], g_ref, rtol=1e-11, atol=1e-11 * np.abs(g_ref).max())
        assert buf[-1] == pytest.approx(ll, rel=1e-12)


def _xc_worker(rank, world, port, q):
    """POINTS_XC algebra with the oracle's per-net passes, 2 chains over 2 ranks:
    rank r runs the branch for chain r on ALL conditions and the trunk for both chains on its
    points; B all-gathered by chain; residuals of both chains at its points; dB of both chains
    reduce-scattered by chain; the branch backward of its chain, the trunk backward of both; the
    all-reduce of [g_lik, sum r^2] per chain == the full-batch values."""
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import network as onet
    arch, prob = _xb_case()
    sh, n_global = pdist.shard_points_xc(prob, rank, world)
    thetas = [prob.frozen.astype(np.float64) + 0.01 * (c + 1) for c in range(world)]   # chain c's parameters
    _, b0, _ = onet.layer_table(arch)
    s2 = prob.noise_sigma ** 2
    Bown, tb = onet.net_forward(arch, thetas[rank], 0, sh.u.astype(np.float64))   # chain = rank, all conditions
    parts = [torch.zeros_like(torch.as_tensor(Bown)) for _ in range(world)]
    dist.all_gather(parts, torch.as_tensor(Bown))                                   # B of every chain
    bufs = []
    dB_parts = []
    tapes_t = []
    Es = []
    for c in range(world):
        T, tt = onet.net_forward(arch, thetas[c], 1, sh.q.astype(np.float64))
        Ball = parts[c].numpy()
        R = sh.v.astype(np.float64) - (Ball @ T.T + thetas[c][b0])
        E = R / s2
        Es.append((E, R, Ball, tt))
        dB_parts.append(torch.as_tensor(E @ T))                  # chain c, all conditions, own points
    dB_own = torch.zeros_like(dB_parts[0])
    dist.reduce_scatter(dB_own, dB_parts)                         # chain block (= rank) gets its full dB
    for c in range(world):
        E, R, Ball, tt = Es[c]
        g = np.zeros_like(thetas[c])
        if c == rank:
            onet.net_backward(arch, thetas[c], 0, tb, dB_own.numpy(), g)    # branch: own chain only
        onet.net_backward(arch, thetas[c], 1, tt, E.T @ Ball, g)          # trunk: every chain, own points
        g[b0] += E.sum()
        bufs.append(np.concatenate([g, [-np.sum(R * R) / (2 * s2)]]))
    buf = torch.tensor(np.stack(bufs), dtype=torch.float64)
    dist.all_reduce(buf)
    q.put((rank, buf.numpy(), n_global))
    dist.destroy_process_group()


def test_points_xc_exchange_matches_full_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_xc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import network as onet
    arch, prob = _xb_case()
    data = {"u": prob.u.astype(np.float64), "q": prob.q.astype(np.float64), "v": prob.v.astype(np.float64)}
    for rank, buf, n_global in res:
        assert n_global == 12 * 9
        for c in range(2):
            th = prob.frozen.astype(np.float64) + 0.01 * (c + 1)
            ll, g_ref, _ = onet.loglik_grad(arch, th, data, prob.noise_sigma)
            np.testing.assert_allclose(buf[c, :-1], g_ref, rtol=1e-11, atol=1e-11 * np.abs(g_ref).max())
            assert buf[c, -1] == pytest.approx(ll, rel=1e-12)
