"""Solver configuration, step state, trace recorder and the scalar rules.

``SolverConfig`` has exactly the reference's fields, defaults and validation
(pdhg.py:43-75) so ``asdict(config)`` echoes the same keys.  The scalar rules
(``primal_weight_update``, ``should_restart``, ``default_stepsize``,
``adaptive_stepsize``'s halving rule) are exposed with the reference
signatures for callers and tests; inside ``solve`` the same rules run on the
device in the controller (csrc/finalize.cu).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

FIXED_BETA = "fixed"
ADAPTIVE = "adaptive"
RELATIVE = "relative"
ABSOLUTE = "absolute"

STEP_GROWTH = 1.05   # pdhg.py:39
MAX_HALVINGS = 80    # pdhg.py:40


@dataclass
class SolverConfig:
    tol: float = 1e-4
    time_limit_s: float = 3600.0
    restart_mode: str = ADAPTIVE
    beta: float = 0.5
    beta_sufficient: float = 0.1
    beta_necessary: float = 0.9
    beta_artificial: float = 0.36
    theta: float = 0.5
    eps_zero: float = 1e-10
    max_iters: int = 1_000_000
    deterministic: bool = False
    kkt_mode: str = RELATIVE
    kkt_stride: int = 1
    eta0: float | None = None
    omega0: float = 1.0

    def __post_init__(self):
        # same checks and messages as pdhg.py:61-75
        if self.tol <= 0 or self.time_limit_s <= 0 or self.max_iters < 1:
            raise ValueError("tol, time_limit_s and max_iters must be positive")
        if not 0.0 < self.beta < 1.0:
            raise ValueError("beta must lie in (0, 1)")
        if not 0.0 < self.beta_sufficient < self.beta_necessary < 1.0:
            raise ValueError("need 0 < beta_sufficient < beta_necessary < 1")
        if self.restart_mode not in (FIXED_BETA, ADAPTIVE):
            raise ValueError(f"unknown restart mode {self.restart_mode!r}")
        if self.kkt_mode not in (RELATIVE, ABSOLUTE):
            raise ValueError(f"unknown kkt mode {self.kkt_mode!r}")
        if self.kkt_stride < 1:
            raise ValueError("kkt_stride must be >= 1")
        if self.omega0 <= 0 or (self.eta0 is not None and self.eta0 <= 0):
            raise ValueError("step parameters must be positive")


@dataclass
class StepState:
    """Step-size scale eta and primal weight omega; tau * sigma == eta ** 2."""

    eta: float
    omega: float

    @property
    def tau(self) -> float:
        return self.eta / self.omega

    @property
    def sigma(self) -> float:
        return self.eta * self.omega


@dataclass
class SolveTrace:
    """Optional per-run recordings (pdhg.py:106-118).  Recording snapshots
    (restart_points, record_inner) makes solve() advance pass by pass."""

    record_inner: bool = False
    etas: list = field(default_factory=list)
    step_bounds: list = field(default_factory=list)
    candidate_kkts: list = field(default_factory=list)
    omegas: list = field(default_factory=list)
    restart_points: list = field(default_factory=list)
    restart_kkts: list = field(default_factory=list)
    inner_iterates: list = field(default_factory=list)
    inner_averages: list = field(default_factory=list)


def default_stepsize(prob) -> float:
    """1 / (2 sqrt(m + n)), half the inverse operator norm (pdhg.py:225-227)."""
    return 1.0 / (2.0 * math.sqrt(prob.m + prob.n))


def primal_weight_update(delta_X: float, delta_pq: float, omega_prev: float, theta: float = 0.5,
                         eps_zero: float = 1e-10) -> float:
    """Log-space smoothing of the dual/primal progress ratio (pdhg.py:174-186)."""
    if omega_prev <= 0:
        raise ValueError("omega_prev must be positive")
    if delta_X > eps_zero and delta_pq > eps_zero:
        return math.exp(theta * math.log(delta_pq / delta_X) + (1.0 - theta) * math.log(omega_prev))
    return omega_prev


def should_restart(config: SolverConfig, candidate_kkt: float, epoch_start_kkt: float,
                   prev_candidate_kkt: float, k: int, total_iterations: int) -> bool:
    """Restart test (pdhg.py:198-222); the device controller applies the same rule."""
    if config.restart_mode == FIXED_BETA:
        return candidate_kkt <= config.beta * epoch_start_kkt
    if candidate_kkt <= config.beta_sufficient * epoch_start_kkt:
        return True
    if candidate_kkt <= config.beta_necessary * epoch_start_kkt and candidate_kkt > prev_candidate_kkt:
        return True
    return k >= config.beta_artificial * total_iterations


def eta_from_bound(bound: float, eta_current: float) -> float:
    """The halving/growth rule of adaptive_stepsize (pdhg.py:166-171)."""
    if math.isinf(bound):
        return eta_current
    eta = eta_current
    while eta > bound:
        eta *= 0.5
    return min(STEP_GROWTH * eta, bound)
