"""fp64 CPU oracle for the VI-informed subset HMC hot path (arXiv 2507.14652).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` leg / `--impl reference` arm may import, call or execute anything under
`oracle/`.  The product path (`paper_2507_14652_b200/`) never imports it and shares no
code with it (no kernels, helpers, constants or table generators); the only common
dependency is the seeded input generator package `hmcdata/`, which holds none of the
method's arithmetic.

Plain, slow, obviously-correct NumPy float64 implementation of:
  network.py  - parameter layout, forward (MLP / DeepONet) and hand-written reverse mode
  philox.py   - Philox4x32-10 counter RNG, uniforms and Box-Muller normals
  hmc.py      - reduced-space log-posterior + gradient (Algorithm 2 target), momentum
                draw, kick-drift-kick leapfrog, Metropolis-Hastings step, chains
  sensitivity.py - parameter sensitivities S_i^2 (eqn:sensitivities) and the tau-partition
                (eqn:threshold) of the step before the hot path
  diagnostics.py - split-R^ and effective sample size (BDA3 §11.4-11.5; NEXT-4)
  (hmc.py also holds the dual-averaging step-size adaptation (NEXT-2) and the posterior
  predictive (NEXT-4))

Each function cites the PAPER.md passage (P:line) or SURVEY.md reading it follows.
Parity status: every function is pinned by a `-m "not gpu"` test in tests/test_oracle_*.py
(closed forms, finite differences, invariants, known answers); see DESIGN.md §4.
"""
from . import network, philox, hmc, sensitivity, diagnostics  # noqa: F401
