"""Value types of the solver API: Iterate, KKTReport, SolveReport.

Field names and semantics follow the reference records (kkt.py:21-53,
reports.py:9-38) so callers and JSON consumers see the same shapes.
"""

from __future__ import annotations

import json
from dataclasses import asdict, dataclass, field

import numpy as np


@dataclass(eq=False)
class Iterate:
    """Primal plan X (m x n) and dual vectors p (m), q (n) as numpy arrays."""

    X: np.ndarray
    p: np.ndarray
    q: np.ndarray

    @classmethod
    def zeros(cls, m: int, n: int) -> "Iterate":
        return cls(np.zeros((m, n)), np.zeros(m), np.zeros(n))

    def copy(self) -> "Iterate":
        return Iterate(self.X.copy(), self.p.copy(), self.q.copy())

    def norm(self) -> float:
        """Euclidean norm of the stacked (vec X, p, q) (host helper)."""
        return float(np.sqrt(np.vdot(self.X, self.X) + np.vdot(self.p, self.p) + np.vdot(self.q, self.q)))


@dataclass(eq=False)
class KKTReport:
    primal_row: np.ndarray      # X 1 - f
    primal_col: np.ndarray      # X^T 1 - g
    dual_violation: np.ndarray  # [p 1^T + 1 q^T - C]^+
    gap: float                  # <C, X> - f.p - g.q
    scale_R: float
    composite: float
    relative_composite: float


@dataclass
class SolveReport:
    """Per-solve record; identical fields to the reference SolveReport."""

    method: str
    solved: bool
    wall_time_s: float
    iterations: int
    restarts: int
    final_relative_kkt: float
    rounded_objective: float
    duality_gap: float
    termination_reason: str
    config_echo: dict = field(default_factory=dict)
    restart_lengths: list = field(default_factory=list)
    restart_kkts: list = field(default_factory=list)

    def to_json(self) -> str:
        return json.dumps(asdict(self), indent=2, sort_keys=True)

    @classmethod
    def from_json(cls, text: str) -> "SolveReport":
        return cls(**json.loads(text))
