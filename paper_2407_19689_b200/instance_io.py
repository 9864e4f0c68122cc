"""Plain-text instance files, compatible with the reference's format
(instance.py:255-333): ``m n`` / ``cost <l1|l2|linf|explicit>`` / m cost rows
when explicit / one line of f / one line of g; ``#`` lines are comments.
Grid-tagged costs are written as the one-line shorthand only when the entries
equal the canonical grid cost."""

from __future__ import annotations

import math

import numpy as np

from .instances import (GRID_KINDS, CostMatrix, InstanceError, Marginal, OTProblem, grid_cost)

KINDS = GRID_KINDS + ("explicit",)


class InstanceFormatError(InstanceError):
    """Malformed instance file (instance.py:31-32)."""


def _fmt(v) -> str:
    return " ".join(str(x) for x in np.asarray(v).tolist())


def _canonical_grid(prob) -> bool:
    kind = getattr(getattr(prob, "cost", None), "norm_kind", "explicit")
    if kind == "explicit" or prob.m != prob.n:
        return False
    r = math.isqrt(prob.m)
    return r * r == prob.m and np.array_equal(prob.C, grid_cost(r, kind).entries)


def save_instance(prob, path) -> None:
    if _canonical_grid(prob):
        lines = ["# otsolve instance", f"{prob.m} {prob.n}", f"cost {prob.cost.norm_kind}"]
    else:
        lines = ["# otsolve instance", f"{prob.m} {prob.n}", "cost explicit"]
        lines.extend(_fmt(row) for row in prob.C)
    lines.append(_fmt(prob.f))
    lines.append(_fmt(prob.g))
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("\n".join(lines) + "\n")


def _floats(tokens, count, what):
    if len(tokens) != count:
        raise InstanceFormatError(f"dimension mismatch in {what}")
    try:
        return np.array([float(t) for t in tokens], dtype=np.float64)
    except ValueError as exc:
        raise InstanceFormatError(f"could not parse {what}: {exc}") from exc


def load_instance(path) -> OTProblem:
    with open(path, "r", encoding="utf-8") as fh:
        lines = [ln.strip() for ln in fh]
    lines = [ln for ln in lines if ln and not ln.startswith("#")]
    if len(lines) < 4:
        raise InstanceFormatError("instance file is truncated")
    dims = lines[0].split()
    if len(dims) != 2:
        raise InstanceFormatError("first line must be 'm n'")
    try:
        m, n = int(dims[0]), int(dims[1])
    except ValueError as exc:
        raise InstanceFormatError(f"could not parse dimensions: {exc}") from exc
    if m < 1 or n < 1:
        raise InstanceFormatError("dimensions must be positive")
    head = lines[1].split()
    if len(head) != 2 or head[0] != "cost":
        raise InstanceFormatError("second line must be 'cost <kind>'")
    kind = head[1]
    if kind not in KINDS:
        raise InstanceFormatError(f"unknown cost kind {kind!r}")
    pos = 2
    if kind == "explicit":
        if len(lines) < 2 + m + 2:
            raise InstanceFormatError("instance file is truncated")
        cost = CostMatrix(np.stack([_floats(lines[pos + i].split(), n, f"cost row {i}") for i in range(m)]),
                          "explicit")
        pos += m
    else:
        if m != n:
            raise InstanceFormatError("grid cost requires m == n")
        r = math.isqrt(m)
        if r * r != m:
            raise InstanceFormatError("grid cost requires a perfect-square dimension")
        cost = grid_cost(r, kind)
    if len(lines) != pos + 2:
        raise InstanceFormatError("instance file has trailing or missing lines")
    f = _floats(lines[pos].split(), m, "row marginal")
    g = _floats(lines[pos + 1].split(), n, "column marginal")
    return OTProblem(cost, Marginal(f), Marginal(g))
