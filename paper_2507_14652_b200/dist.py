"""Multi-GPU plumbing for the hot path (one process per GPU, torch.distributed for setup only).

- chain mode: each rank runs its own chains (global chain ids key Philox); no data-path
  collective.  `chain_ids(rank, C)`.
- data mode: the training set is sharded by rows (MLP: rows of x/y; DeepONet: condition rows
  of u/v, trunk inputs replicated - or, unaligned, the same rows of the per-pair q); libhmc all-reduces [g_lik, sum r^2] in-graph with NCCL each
  leapfrog step and adds the prior once after the reduction.  `shard_rows` cuts
  this rank's block; `shard_points_xb` the POINTS_XB condition x point blocks (DeepONet: the
  branch outputs are all-gathered and dB reduce-scattered in-graph); `broadcast_nccl_id` ships rank 0's NCCL unique id over the process group.
Marshalling only: no arithmetic of the method lives here.
"""
from __future__ import annotations

import copy

import numpy as np


def chain_ids(rank: int, n_chains: int) -> np.ndarray:
    return (rank * n_chains + np.arange(n_chains)).astype(np.uint32)


def row_block(n: int, rank: int, world: int):
    """Contiguous, near-equal row block [lo, hi) of rank (first n % world ranks get one more)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_rows(problem, rank: int, world: int):
    """Copy of `problem` holding only this rank's row block of the data; returns (shard, n_global)."""
    sh = copy.copy(problem)
    if problem.arch.kind == "mlp":
        n = problem.x.shape[0]
        lo, hi = row_block(n, rank, world)
        sh.x = np.ascontiguousarray(problem.x[lo:hi])
        sh.y = np.ascontiguousarray(problem.y[lo:hi])
        return sh, n
    n_c, n_x = problem.v.shape
    lo, hi = row_block(n_c, rank, world)
    sh.u = np.ascontiguousarray(problem.u[lo:hi])
    sh.v = np.ascontiguousarray(problem.v[lo:hi])
    if np.asarray(problem.q).ndim == 3:  # unaligned DeepONet: each function's own query points
        sh.q = np.ascontiguousarray(problem.q[lo:hi])
    return sh, n_c * n_x


def shard_points_xb(problem, rank: int, world: int):
    """POINTS_XB layout (DeepONet with shared query points): condition block r of u
    (n_c / world rows, n_c divisible by world), point block r of q, and v for ALL conditions at
    those points.  Returns (shard, n_global)."""
    n_c, n_x = problem.v.shape
    assert n_c % world == 0, "POINTS_XB needs n_c divisible by world"
    c0, c1 = row_block(n_c, rank, world)
    x0, x1 = row_block(n_x, rank, world)
    sh = copy.copy(problem)
    sh.u = np.ascontiguousarray(problem.u[c0:c1])
    sh.q = np.ascontiguousarray(problem.q[x0:x1])
    sh.v = np.ascontiguousarray(problem.v[:, x0:x1])
    return sh, n_c * n_x


def shard_points_xc(problem, rank: int, world: int):
    """POINTS_XC layout (DeepONet with shared query points): ALL conditions of u (the
    branch runs this rank's chain block on all of them), point block r of q, and v for all
    conditions at those points.  Returns (shard, n_global)."""
    n_c, n_x = problem.v.shape
    x0, x1 = row_block(n_x, rank, world)
    sh = copy.copy(problem)
    sh.q = np.ascontiguousarray(problem.q[x0:x1])
    sh.v = np.ascontiguousarray(problem.v[:, x0:x1])
    return sh, n_c * n_x


def broadcast_nccl_id(make_id, group=None) -> bytes:
    """Rank 0 calls make_id() (libhmc's hmc_comm_unique_id); every rank returns the same bytes."""
    import torch.distributed as dist
    obj = [make_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def make_context(problem, mode: str, rank: int, world: int, group=None, shard: str = "rows"):
    """libhmc context for this rank: 'chain' (own chains) or 'data' (row shard, or the POINTS_XB
    condition x point blocks, + NCCL)."""
    from . import abi
    C = problem.n_chains
    if mode == "chain" or (world == 1 and shard == "rows"):
        return abi.Context(problem, mode="chain" if world > 1 else "single", rank=rank, world=world,
                           chain_ids=chain_ids(rank, C) if world > 1 else None)
    if shard == "points_xb":
        sh, n_global = shard_points_xb(problem, rank, world)
    elif shard == "points_xc":
        sh, n_global = shard_points_xc(problem, rank, world)
    else:
        sh, n_global = shard_rows(problem, rank, world)
    nid = broadcast_nccl_id(abi.hmc_comm_unique_id, group) if world > 1 else None
    return abi.Context(sh, mode="data", rank=rank, world=world, nccl_id=nid, n_global=n_global, shard=shard)
