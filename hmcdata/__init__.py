"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds ONLY input generation (data, frozen VI means, VI sigmas,
active-index masks) and the config table of BASELINE.json / SURVEY.md §8.
It contains none of the method's arithmetic (no log-posterior, gradient,
leapfrog, Metropolis or RNG of the sampler); both `oracle/` and
`paper_2507_14652_b200/` consume its arrays and neither shares code with the
other.
"""
from .configs import ArchSpec, NetSpec, Problem, CONFIGS, config_names  # noqa: F401
from .generate import make_problem, make_tiny_problem  # noqa: F401
