"""Block screening of the STEP pass (csrc/screen.cu) must not change a single bit.

A screened pass skips 8x16 cells whose every output and reduction term is
exactly +0 (zero plan and lagged average there, no dual violation by the
current or averaged duals), so solves with screening on and off must agree
bit for bit: reports, iterates (compared as int64 bit patterns, so -0.0 and
+0.0 differ), traces.  The dense TMA walker is the reference here; its own
parity with the oracle is covered by test_gpu_solve / test_gpu_units.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture
def pd():
    import paper_2407_19689_b200 as pd
    from paper_2407_19689_b200 import device
    yield pd
    device.set_screening(None)


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)


def _same_iterate(a, b):
    return (np.array_equal(_bits(a.X), _bits(b.X)) and np.array_equal(_bits(a.p), _bits(b.p))
            and np.array_equal(_bits(a.q), _bits(b.q)))


def _solve_both(pd, prob, cfg, initial=None, trace=False):
    from paper_2407_19689_b200 import device
    out = []
    for on in (False, True):
        device.set_screening(on)
        tr = pd.SolveTrace(record_inner=trace) if trace else None
        it, rep = pd.solve(prob, cfg, initial=initial, trace=tr)
        out.append((it, rep, tr))
    return out


def _raw(C, f, g):
    from types import SimpleNamespace
    return SimpleNamespace(C=C, f=f, g=g, m=C.shape[0], n=C.shape[1], cost_fro_norm=float(np.linalg.norm(C)),
                           marginal_norm=float(np.linalg.norm(f) + np.linalg.norm(g)))


def _random_problem(m, n, seed):
    rng = np.random.default_rng(seed)
    C = rng.random((m, n))
    f = rng.random(m) + 0.1
    g = rng.random(n) + 0.1
    return _raw(C, f / f.sum(), g / g.sum())


CASES = [
    ("sqeuclid_r8", lambda inst: inst.sqeuclid_problem(8, 1), dict(tol=1e-6)),
    ("sqeuclid_r16", lambda inst: inst.sqeuclid_problem(16, 0), dict(tol=1e-5)),
    ("c1_seed0", lambda inst: inst.sqeuclid_problem(32, 0), dict(tol=1e-4)),
    ("l1_grid_r16", lambda inst: inst.grid_problem("whitenoise", 16, "l1", 3), dict(tol=1e-5)),
    ("rect_sparse", lambda inst: inst.rect_problem(2, src_shape=(8, 16), dst_shape=(16, 32)), dict(tol=1e-5)),
    ("random_37x53", lambda inst: _random_problem(37, 53, 4), dict(tol=1e-6)),
    ("random_1x9", lambda inst: _random_problem(1, 9, 5), dict(tol=1e-7)),
    ("random_9x1", lambda inst: _random_problem(9, 1, 6), dict(tol=1e-7)),
    ("fixed_mode", lambda inst: inst.sqeuclid_problem(8, 2), dict(tol=1e-5, restart_mode="fixed")),
    ("stride_abs", lambda inst: inst.sqeuclid_problem(8, 3), dict(tol=1e-5, kkt_stride=3, kkt_mode="absolute")),
    ("iter_limit", lambda inst: inst.sqeuclid_problem(16, 4), dict(tol=1e-9, max_iters=150)),
]


@pytest.mark.parametrize("name,make,kw", CASES, ids=[c[0] for c in CASES])
def test_screened_solve_bit_identical(pd, name, make, kw):
    from paper_2407_19689_b200 import instances as inst
    prob = make(inst)
    cfg = pd.SolverConfig(deterministic=True, **kw)
    (it0, r0, _), (it1, r1, _) = _solve_both(pd, prob, cfg)
    assert r0.to_json() == r1.to_json(), name
    assert _same_iterate(it0, it1), name


def test_screened_warm_start_and_trace(pd):
    """Warm start from a dense random plan (every cell occupied at first) and
    the stepwise trace path (snapshots of every iterate and average)."""
    from paper_2407_19689_b200 import instances as inst
    prob = inst.sqeuclid_problem(8, 5)
    rng = np.random.default_rng(7)
    init = pd.Iterate(rng.random((64, 64)) * 1e-3, rng.standard_normal(64) * 0.01, rng.standard_normal(64) * 0.01)
    cfg = pd.SolverConfig(tol=1e-5, deterministic=True)
    (it0, r0, t0), (it1, r1, t1) = _solve_both(pd, prob, cfg, initial=init, trace=True)
    assert r0.to_json() == r1.to_json()
    assert _same_iterate(it0, it1)
    assert len(t0.inner_iterates) == len(t1.inner_iterates) == r0.iterations
    for a, b in zip(t0.inner_iterates + t0.inner_averages + t0.restart_points,
                    t1.inner_iterates + t1.inner_averages + t1.restart_points):
        assert _same_iterate(a, b)


@pytest.mark.parametrize("blocks", [1, 3])
def test_screened_k0_many_tiles_per_warp(pd, monkeypatch, blocks):
    """K0 is persistent: each warp walks tiles warp, warp + nw, ...  Capping its
    grid (PDOT_K0_BLOCKS) gives every warp 32 or 11 tiles of a 4096^2 warm start
    from a dense plan (every tile occupied, so every tile takes the per-cell
    screen): still bit-identical to the dense walker."""
    from paper_2407_19689_b200 import instances as inst
    monkeypatch.setenv("PDOT_K0_BLOCKS", str(blocks))
    prob = inst.sqeuclid_problem(64, 2)  # 4096^2: 256 tiles of 128 x 512
    n = prob.m
    rng = np.random.default_rng(11)
    X0 = rng.random((n, n)) * 1e-9
    X0[rng.random((n, n)) < 0.5] = 0.0
    init = pd.Iterate(X0, rng.standard_normal(n) * 1e-3, rng.standard_normal(n) * 1e-3)
    cfg = pd.SolverConfig(tol=1e-9, max_iters=40, deterministic=True)
    (it0, r0, _), (it1, r1, _) = _solve_both(pd, prob, cfg, initial=init)
    assert r0.to_json() == r1.to_json()
    assert _same_iterate(it0, it1)


def test_screened_implicit_cost(pd):
    prob = pd.DeviceProblem.sqeuclid_grid(32, 2, implicit=True)
    cfg = pd.SolverConfig(tol=1e-4, deterministic=True)
    (it0, r0, _), (it1, r1, _) = _solve_both(pd, prob, cfg)
    assert r0.to_json() == r1.to_json()
    assert _same_iterate(it0, it1)


@pytest.mark.parametrize("k", [0, 3])
def test_screened_unit_step(pd, k):
    """pdhg_step (and the averaged unit step) through the screened walker, on a
    sparse plan and on a dense one, against the dense walker."""
    from paper_2407_19689_b200 import device, instances as inst, units
    prob = inst.sqeuclid_problem(8, 1)
    rng = np.random.default_rng(3)
    X = np.zeros((64, 64))
    X[rng.integers(0, 64, 40), rng.integers(0, 64, 40)] = rng.random(40)
    for plan in (X, rng.random((64, 64))):
        it = pd.Iterate(plan, rng.standard_normal(64) * 5, rng.standard_normal(64) * 5)
        res = []
        for on in (False, True):
            device.set_screening(on)
            if k:
                avg = pd.Iterate(plan * 0.5, it.p * 0.3, it.q * 0.3)
                res.append(units.step_and_average(prob, it, avg, 0.01, 0.5, k))
            else:
                res.append(pd.pdhg_step(prob, it, 0.01, 0.5))
        if k:
            (n0, a0), (n1, a1) = res
            assert _same_iterate(n0, n1) and _same_iterate(a0, a1)
        else:
            assert _same_iterate(res[0], res[1])


def test_screening_engages(pd):
    """At C1 the screened passes must touch a small part of the plan."""
    from paper_2407_19689_b200 import device
    device.set_screening(True)
    dp = pd.DeviceProblem.sqeuclid_grid(32, 0)
    h = device.get_handle(dp.m, dp.n, dp.device)
    h.bind(dp)
    h.screen_stats(reset=True)
    _, rep = pd.solve(dp, pd.SolverConfig(tol=1e-4, deterministic=True))
    st = h.screen_stats()
    assert st["screen_on"] == 1
    assert st["passes"] >= rep.iterations
    frac = st["active_cells"] / (st["passes"] * st["cells_per_plan"])
    print("C1 active cell fraction", frac, st)
    assert frac < 0.3


@pytest.mark.parametrize("bad", [np.inf, np.nan])
def test_screened_non_finite_costs(pd, bad):
    """Non-finite costs: their cells (and tiles) are never screened out (min C =
    -inf), so whatever the dense walker does with inf * 0 or NaN -- a result or
    the same exception -- the screened walker reproduces it."""
    from paper_2407_19689_b200 import instances as inst
    base = inst.sqeuclid_problem(32, 6)  # 1024 x 1024: many row and column tiles
    C = np.array(base.C, dtype=np.float64)
    C[700, 37] = bad
    C[5, 1000] = bad
    prob = _raw(C, np.asarray(base.f), np.asarray(base.g))
    cfg = pd.SolverConfig(tol=1e-4, deterministic=True, max_iters=60)
    out = []
    from paper_2407_19689_b200 import device
    for on in (False, True):
        device.set_screening(on)
        try:
            it, rep = pd.solve(prob, cfg)
            out.append(("ok", rep.to_json(), it))
        except Exception as e:  # noqa: BLE001 - the same failure is the expectation
            out.append(("err", type(e).__name__ + str(e), None))
    assert out[0][0] == out[1][0] and out[0][1] == out[1][1]
    if out[0][0] == "ok":
        assert _same_iterate(out[0][2], out[1][2])


def test_screened_far_violation(pd):
    """A single cell far from the support whose cost is low enough to be
    violated: the tile-level screen must keep its tile and the cell screen must
    catch it."""
    from paper_2407_19689_b200 import instances as inst
    base = inst.sqeuclid_problem(32, 7)
    C = np.array(base.C, dtype=np.float64)
    C[900, 40] = -5.0  # far off the diagonal, strongly attractive
    prob = _raw(C, np.asarray(base.f), np.asarray(base.g))
    cfg = pd.SolverConfig(tol=1e-4, deterministic=True, max_iters=400)
    (it0, r0, _), (it1, r1, _) = _solve_both(pd, prob, cfg)
    assert r0.to_json() == r1.to_json()
    assert _same_iterate(it0, it1)


def test_screened_wide_rows_beyond_4096_cells(pd):
    """n > 65536: a row of 8x16 cells has more than 4096 cells, so the cell
    index of a 32-bit list entry needs more than 12 bits (the band takes the
    remaining bits, csrc/pdot_internal.cuh cell_entry).  80 x 65552 is above
    2^22 entries, so screening is the default: it must be on, and agree bit for
    bit with the dense walker, including the sparse device->host copy of the
    final plan."""
    from paper_2407_19689_b200 import instances as inst
    from paper_2407_19689_b200.device import get_handle
    m, n = 80, 65552
    rng = np.random.default_rng(3)
    # a sparse-plan problem: L1-like cost between row and column coordinates
    a = np.sort(rng.random(m)) * n
    C = np.abs(a[:, None] - np.arange(n)[None, :]) / 100.0
    f = rng.random(m) + 0.1
    g = rng.random(n) + 0.1
    prob = inst.make_problem(C, f, g)
    cfg = pd.SolverConfig(tol=1e-9, deterministic=True, max_iters=80)
    (it0, r0, _), (it1, r1, _) = _solve_both(pd, prob, cfg)
    assert get_handle(m, n).screened()
    assert r0.to_json() == r1.to_json()
    assert _same_iterate(it0, it1)
    assert np.count_nonzero(it1.X[:, 65536:]) > 0  # cells past index 4095 carry mass


def test_c5_geometry_virtual_shards(pd):
    """C5 geometry (n = 65536, the widest row of cells a 12-bit index held) on a
    reduced row count: rows 0..1023 of the 65536^2 instance, generated on the
    device, solved on one handle and as 8 virtual row shards (screened passes,
    device-copy exchange): bit-identical."""
    from paper_2407_19689_b200.shard import solve_virtual
    dp = pd.DeviceProblem.sqeuclid_grid(256, 0, rows=(0, 1024))
    cfg = pd.SolverConfig(tol=1e-9, deterministic=True, max_iters=40)
    it1, rep1 = pd.solve(dp, cfg)
    assert pd.device.get_handle(dp.m, dp.n).screened()
    itv, repv = solve_virtual(dp, cfg, 8)
    assert (repv.iterations, repv.restarts, repv.restart_lengths) == (rep1.iterations, rep1.restarts,
                                                                       rep1.restart_lengths)
    assert repv.final_relative_kkt == rep1.final_relative_kkt
    assert np.array_equal(itv.X, it1.X) and np.array_equal(itv.p, it1.p) and np.array_equal(itv.q, it1.q)
