"""Philox4x32-10 counter-based RNG in vectorised NumPy uint64.  TEST INFRASTRUCTURE ONLY.

The paper draws p ~ N(0, M) (Algorithm 1/2) and u ~ U[0,1]
without naming a generator.  Reading: Philox4x32-10 with
key (k0, k1) = (seed mod 2^32, seed >> 32) and counter (c0, c1, c2, c3) =
(j >> 2, tag, iter, chain_id); tag 0 = momentum, 1 = MH uniform, 2 = init jitter.
Round: (hi0, lo0) = mulhilo(0xD2511F53, c0); (hi1, lo1) = mulhilo(0xCD9E8D57, c2);
c <- (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0); key += (0x9E3779B9, 0xBB67AE85) between
rounds.  Uniform u = (x + 0.5) 2^-32 in fp64; Box-Muller on (u0,u1) and (u2,u3).
"""
from __future__ import annotations

import numpy as np

MASK = np.uint64(0xFFFFFFFF)
M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = np.uint64(0x9E3779B9)
W1 = np.uint64(0xBB67AE85)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised over counters; all args broadcastable integer arrays (< 2^32)."""
    c0, c1, c2, c3 = (np.asarray(a, dtype=np.uint64) & MASK for a in (c0, c1, c2, c3))
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    c0, c1, c2, c3 = (a.copy() for a in (c0, c1, c2, c3))
    k0 = np.uint64(int(k0) & 0xFFFFFFFF)
    k1 = np.uint64(int(k1) & 0xFFFFFFFF)
    for r in range(10):
        p0 = M0 * c0                      # < 2^64, exact in uint64
        p1 = M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0), lo1, (hi0 ^ c3 ^ k1), lo0
        if r < 9:
            k0 = (k0 + W0) & MASK
            k1 = (k1 + W1) & MASK
    return c0, c1, c2, c3


def _key(seed):
    seed = int(seed)
    return seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF


def uniform01(x):
    """u = (x + 0.5) * 2^-32 in fp64, strictly inside (0, 1)."""
    return (np.asarray(x, dtype=np.float64) + 0.5) * (2.0 ** -32)


def normals(seed, tag, it, chain, n):
    """z_j for j < n: counter (j>>2, tag, iter, chain), lane j & 3, Box-Muller in fp64."""
    k0, k1 = _key(seed)
    blocks = (n + 3) // 4
    x0, x1, x2, x3 = philox4x32_10(np.arange(blocks), tag, it, chain, k0, k1)
    u0, u1, u2, u3 = (uniform01(a) for a in (x0, x1, x2, x3))
    r01 = np.sqrt(-2.0 * np.log(u0))
    r23 = np.sqrt(-2.0 * np.log(u2))
    z = np.stack([r01 * np.cos(2.0 * np.pi * u1), r01 * np.sin(2.0 * np.pi * u1),
                  r23 * np.cos(2.0 * np.pi * u3), r23 * np.sin(2.0 * np.pi * u3)], axis=1)
    return z.reshape(-1)[:n]


def mh_uniform(seed, it, chain):
    """u ~ U(0,1) of the Metropolis step: tag 1, counter (0, 1, iter, chain), word 0."""
    k0, k1 = _key(seed)
    x0, _, _, _ = philox4x32_10(0, 1, it, chain, k0, k1)
    return float(uniform01(x0))


def words(seed, tag, it, chain, nblocks):
    """Raw 32-bit words, block-major (for the bitwise GPU agreement test)."""
    k0, k1 = _key(seed)
    x = philox4x32_10(np.arange(nblocks), tag, it, chain, k0, k1)
    return np.stack(x, axis=1).astype(np.uint32)
