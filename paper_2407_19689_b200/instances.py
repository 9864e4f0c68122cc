"""Problem containers and the synthetic instance families of BASELINE.json.

The solver consumes any object exposing ``C f g m n cost_fro_norm
marginal_norm`` (the accessors of the reference ``OTProblem``,
instance.py:109-150), so a reference ``otsolve.OTProblem`` can be passed in
unchanged.  This module provides a minimal equivalent for callers that do not
have the reference installed, plus the generators for the benchmark configs
(SURVEY.md §8(d)):

* ``sqeuclid_grid_cost(r)`` — squared Euclidean grid cost as EXACT integers
  ``di^2 + dj^2`` (``grid_cost('l2')**2`` rounds through sqrt).
* ``whitenoise_marginals(r, seed)`` — the reference ``synth_instance(
  "whitenoise", r, seed)`` + ``marginal_from_image`` (instance.py:350-351,
  369-376, 300-305, 78-82), restated.
* ``rect_l1_cost`` / ``sparse_marginals`` — the builder-defined rectangular
  C4 family.

The on-device twins of the cost generators live in the CUDA library
(``pdot_gen_cost``); both produce integers, so they agree bit for bit.
"""

from __future__ import annotations

import math

import numpy as np


class InstanceError(ValueError):
    """Invalid instance data (mirrors instance.py:28-29)."""


def _finite(values, name):
    arr = np.array(values, dtype=np.float64)
    if not np.all(np.isfinite(arr)):
        raise InstanceError(f"non-finite {name} entry")
    return arr


class Marginal:
    """Probability vector normalised to unit sum (instance.py:66-85)."""

    def __init__(self, weights):
        w = _finite(weights, "marginal")
        if w.ndim != 1 or w.size < 1:
            raise InstanceError("marginal must be a non-empty vector")
        if np.any(w < 0):
            raise InstanceError("negative marginal entry")
        total = float(w.sum())
        if total <= 0.0:
            raise InstanceError("marginal has zero mass")
        self.weights = w / total

    def __len__(self):
        return self.weights.size


class CostMatrix:
    """Non-negative cost matrix (instance.py:88-106)."""

    def __init__(self, entries, norm_kind="explicit"):
        e = _finite(entries, "cost")
        if e.ndim != 2:
            raise InstanceError("cost must be a 2-D matrix")
        if np.any(e < 0):
            raise InstanceError("negative cost entry")
        self.entries = e
        self.norm_kind = norm_kind

    @property
    def shape(self):
        return self.entries.shape


class OTProblem:
    """Cost + marginals with the accessors the solver reads (instance.py:109-150)."""

    def __init__(self, cost, row_marginal, col_marginal):
        if not isinstance(cost, CostMatrix):
            cost = CostMatrix(cost)
        if not isinstance(row_marginal, Marginal):
            row_marginal = Marginal(row_marginal)
        if not isinstance(col_marginal, Marginal):
            col_marginal = Marginal(col_marginal)
        m, n = cost.shape
        if len(row_marginal) != m or len(col_marginal) != n:
            raise InstanceError("dimension mismatch between cost and marginals")
        self.cost, self.row_marginal, self.col_marginal = cost, row_marginal, col_marginal
        self._fro = None
        self._marg = None

    @property
    def m(self):
        return self.cost.shape[0]

    @property
    def n(self):
        return self.cost.shape[1]

    @property
    def C(self):
        return self.cost.entries

    @property
    def f(self):
        return self.row_marginal.weights

    @property
    def g(self):
        return self.col_marginal.weights

    @property
    def cost_fro_norm(self):
        if self._fro is None:
            self._fro = float(np.linalg.norm(self.C))
        return self._fro

    @property
    def marginal_norm(self):
        if self._marg is None:
            self._marg = float(np.linalg.norm(self.f) + np.linalg.norm(self.g))
        return self._marg


def make_problem(C, f, g):
    return OTProblem(CostMatrix(C), Marginal(f), Marginal(g))


# ---------------------------------------------------------------------------
# benchmark families
# ---------------------------------------------------------------------------
def grid_coords(r):
    """Row-major integer coordinates (k // r, k % r) (instance.py:161-164)."""
    k = np.arange(r * r, dtype=np.int64)
    return k // r, k % r


def sqeuclid_grid_cost(r):
    """Exact squared-Euclidean cost between the cells of an r x r grid."""
    a, b = grid_coords(r)
    da = a[:, None] - a[None, :]
    db = b[:, None] - b[None, :]
    return (da * da + db * db).astype(np.float64)


def sqeuclid_grid_cost_rows(r, row0, row1):
    """Rows [row0, row1) of sqeuclid_grid_cost(r) without building the rest."""
    a, b = grid_coords(r)
    da = a[row0:row1, None] - a[None, :]
    db = b[row0:row1, None] - b[None, :]
    return (da * da + db * db).astype(np.float64)


def l1_grid_cost(r):
    a, b = grid_coords(r)
    return (np.abs(a[:, None] - a[None, :]) + np.abs(b[:, None] - b[None, :])).astype(np.float64)


GRID_KINDS = ("l1", "l2", "linf")
SYNTH_CLASSES = ("whitenoise", "shapes", "cauchy_like")


def grid_cost(r, norm_kind, normalize=False):
    """Pairwise l1 / l2 / linf distances between the cells of an r x r grid
    (restates instance.py:167-191 with the same numpy operations, so the
    entries are bit-identical; l2 goes through sqrt)."""
    if r < 1:
        raise InstanceError("grid resolution must be positive")
    if norm_kind not in GRID_KINDS:
        raise InstanceError(f"grid cost kind must be one of {GRID_KINDS}")
    a, b = grid_coords(r)
    coords = np.stack([a, b], axis=1).astype(np.float64)
    diff = np.abs(coords[:, None, :] - coords[None, :, :])
    if norm_kind == "l1":
        entries = diff.sum(axis=2)
    elif norm_kind == "l2":
        entries = np.sqrt((diff ** 2).sum(axis=2))
    else:
        entries = diff.max(axis=2)
    if normalize and entries.max() > 0:
        entries = entries / entries.max()
    return CostMatrix(entries, norm_kind)


def _rect(rng, rows, cols):
    r0 = int(rng.integers(rows.start, rows.stop))
    r1 = int(rng.integers(r0, rows.stop))
    c0 = int(rng.integers(cols.start, cols.stop))
    c1 = int(rng.integers(c0, cols.stop))
    return r0, r1, c0, c1


def _synth_image(kind, r, rng):
    """One synthetic image (instance.py:208-226), same RNG call sequence."""
    if kind == "whitenoise":
        return rng.random((r, r))
    if kind == "shapes":
        pixels = np.zeros((r, r))
        split = int(rng.integers(1, r))
        for rows in (range(0, split), range(split, r)):
            r0, r1, c0, c1 = _rect(rng, rows, range(0, r))
            pixels[r0:r1 + 1, c0:c1 + 1] = 1.0
        return pixels
    if kind == "cauchy_like":
        center = rng.integers(0, r, size=2)
        ii, jj = np.meshgrid(np.arange(r), np.arange(r), indexing="ij")
        d2 = (ii - center[0]) ** 2 + (jj - center[1]) ** 2
        return 1.0 / (1.0 + d2.astype(np.float64))
    raise InstanceError(f"unknown synthetic class {kind!r}")


def synth_images(kind, r, seed):
    """Deterministic pair of synthetic images (instance.py:222-229)."""
    if kind not in SYNTH_CLASSES:
        raise InstanceError(f"unknown synthetic class {kind!r}")
    if r < 2:
        raise InstanceError("synthetic images need resolution >= 2")
    rng = np.random.default_rng(seed)
    return _synth_image(kind, r, rng), _synth_image(kind, r, rng)


def grid_problem(kind, r, norm_kind, seed):
    """Full grid instance: two synthetic images + grid cost (instance.py:232-239)."""
    src, dst = synth_images(kind, r, seed)
    return OTProblem(grid_cost(r, norm_kind), Marginal(src.ravel()), Marginal(dst.ravel()))


def whitenoise_images(r, seed):
    """synth_instance("whitenoise", r, seed), instance.py:350-351, 369-376."""
    if r < 2:
        raise InstanceError("synthetic images need resolution >= 2")
    rng = np.random.default_rng(seed)
    return rng.random((r, r)), rng.random((r, r))


def whitenoise_marginals(r, seed):
    """The two marginals of synth_instance("whitenoise", r, seed), normalised
    ONCE from the raw pixels as marginal_from_image does (instance.py:153-158).
    Callers that build a problem from these weights must not normalise them a
    second time (w / sum(w) of an already-normalised w moves entries by an ulp):
    pass them as ``Marginal`` objects, not arrays (see sqeuclid_problem)."""
    src, dst = whitenoise_images(r, seed)
    return Marginal(src.ravel()).weights, Marginal(dst.ravel()).weights


def whitenoise_marginal_objects(r, seed):
    """(Marginal, Marginal) built from the raw pixels: marginal_from_image."""
    src, dst = whitenoise_images(r, seed)
    return Marginal(src.ravel()), Marginal(dst.ravel())


def sqeuclid_problem(r, seed):
    """C1/C2/C3/C5 family: whitenoise marginals, exact sq-Euclidean cost.

    Marginals are normalised once, from the raw pixels, exactly like the
    reference's grid_problem / marginal_from_image (instance.py:153-158,
    232-239), so f and g are bitwise the ones DeviceProblem.sqeuclid_grid
    uploads."""
    fm, gm = whitenoise_marginal_objects(r, seed)
    prob = OTProblem(CostMatrix(sqeuclid_grid_cost(r)), fm, gm)
    # the exact integer norm, as the device problem uses: equal to the reference's
    # np.linalg.norm(C) up to r = 64 (tested) and free of BLAS rounding beyond
    prob._fro = sqeuclid_fro_norm(r)
    return prob


RECT_SRC = (64, 128)   # C4 source grid (rows, cols)  -> m = 8192
RECT_DST = (128, 256)  # C4 target grid               -> n = 32768


def rect_l1_cost(src_shape=RECT_SRC, dst_shape=RECT_DST):
    """C4: L1 cost from a source grid scaled by 2 onto the target lattice."""
    sr, sc = src_shape
    tr, tc = dst_shape
    k = np.arange(sr * sc, dtype=np.int64)
    a, b = 2 * (k // sc), 2 * (k % sc)
    l = np.arange(tr * tc, dtype=np.int64)
    c, d = l // tc, l % tc
    return (np.abs(a[:, None] - c[None, :]) + np.abs(b[:, None] - d[None, :])).astype(np.float64)


def rect_l1_cost_rows(row0, row1, src_shape=RECT_SRC, dst_shape=RECT_DST):
    sr, sc = src_shape
    tr, tc = dst_shape
    k = np.arange(row0, row1, dtype=np.int64)
    a, b = 2 * (k // sc), 2 * (k % sc)
    l = np.arange(tr * tc, dtype=np.int64)
    c, d = l // tc, l % tc
    return (np.abs(a[:, None] - c[None, :]) + np.abs(b[:, None] - d[None, :])).astype(np.float64)


def sparse_weights(size, seed, density=0.1):
    """Raw C4 weights: `density` of the cells carry U(0.1, 1.1) mass, the rest 0."""
    rng = np.random.default_rng(seed)
    k = max(1, int(round(density * size)))
    support = rng.choice(size, size=k, replace=False)
    w = np.zeros(size)
    w[support] = 0.1 + rng.random(k)
    return w


def sparse_marginals(size, seed, density=0.1):
    """C4 marginals: sparse_weights normalised once (Marginal)."""
    return Marginal(sparse_weights(size, seed, density)).weights


def rect_problem(seed, src_shape=RECT_SRC, dst_shape=RECT_DST):
    """C4 family; marginals normalised once from the raw weights (the same f, g
    as DeviceProblem.rect_l1)."""
    m = src_shape[0] * src_shape[1]
    n = dst_shape[0] * dst_shape[1]
    fm = Marginal(sparse_weights(m, 2 * seed))
    gm = Marginal(sparse_weights(n, 2 * seed + 1))
    prob = OTProblem(CostMatrix(rect_l1_cost(src_shape, dst_shape)), fm, gm)
    prob._fro = rect_l1_fro_norm(src_shape, dst_shape)
    return prob


def grid_side(mn):
    r = math.isqrt(mn)
    if r * r != mn:
        raise InstanceError("not a square grid size")
    return r


# ---------------------------------------------------------------------------
# exact Frobenius norms of the generated integer costs.  Every GPU count (and
# the host) then sees the same cost_fro_norm, so the KKT normalisers -- and
# with them the whole trajectory -- are independent of the sharding.
# ---------------------------------------------------------------------------
def _pair_power_sums(xs, ys, k):
    """sum over (x in xs, y in ys) of |x - y|**k, exact (Python ints)."""
    return sum(abs(x - y) ** k for x in xs for y in ys)


def sqeuclid_fro_norm(r):
    """||C||_F for C_ij = (a_i-a_j)^2 + (b_i-b_j)^2 on an r x r grid:
    sum = 2 r^2 S4 + 2 S2^2 with S_k = sum_{a,a'} (a-a')^k."""
    axis = range(r)
    s2 = _pair_power_sums(axis, axis, 2)
    s4 = _pair_power_sums(axis, axis, 4)
    total = 2 * r * r * s4 + 2 * s2 * s2
    return math.sqrt(float(total))


def l1_grid_fro_norm(r):
    axis = range(r)
    s1 = _pair_power_sums(axis, axis, 1)
    s2 = _pair_power_sums(axis, axis, 2)
    total = 2 * r * r * s2 + 2 * s1 * s1
    return math.sqrt(float(total))


def rect_l1_fro_norm(src_shape=RECT_SRC, dst_shape=RECT_DST):
    """||C||_F of rect_l1_cost: C = |2 r_s - r_t| + |2 c_s - c_t|."""
    sr, sc = src_shape
    tr, tc = dst_shape
    rows_s = [2 * x for x in range(sr)]
    cols_s = [2 * x for x in range(sc)]
    rows_t, cols_t = range(tr), range(tc)
    dx2 = _pair_power_sums(rows_s, rows_t, 2)
    dy2 = _pair_power_sums(cols_s, cols_t, 2)
    dx1 = _pair_power_sums(rows_s, rows_t, 1)
    dy1 = _pair_power_sums(cols_s, cols_t, 1)
    total = sc * tc * dx2 + sr * tr * dy2 + 2 * dx1 * dy1
    return math.sqrt(float(total))
