"""Soundness of the slack certificates, restated on the host with
the device's rounding: K1's record (every operation rounded down, the warp
minimum truncated to its high word), K2's drift counters (rounded up), K0's
test (rounded down).  Exact rational arithmetic checks the claim the K0 test
relies on: whenever it passes, p_i + q_j < C_ij for every entry of the cell and
both dual pairs, so RN(p_i + q_j) <= C_ij as the coarse bound would certify.
Random dual walks include rejected trials (drift counted, duals unchanged),
restarts (both pairs jump to one of the two input pairs) and steps at the
rounding level, with slack close to zero."""

import math
import random
import struct
from fractions import Fraction as F

import pytest


def rd_add(a, b):
    r = a + b
    if not (math.isfinite(r) and math.isfinite(a) and math.isfinite(b)):
        return r  # inf / NaN: exact in IEEE
    return math.nextafter(r, -math.inf) if F(r) > F(a) + F(b) else r


def ru_add(a, b):
    r = a + b
    if not (math.isfinite(r) and math.isfinite(a) and math.isfinite(b)):
        return r
    return math.nextafter(r, math.inf) if F(r) < F(a) + F(b) else r


def rd_sub(a, b):
    return rd_add(a, -b)


def ru_sub(a, b):
    return ru_add(a, -b)


def max_nan(a, b):  # pdot_internal.cuh max_nan
    return a if (a > b or a != a) else b


def absdiff_ru(a, b):  # pdot_internal.cuh absdiff_ru
    return max_nan(ru_sub(a, b), ru_sub(b, a))


def hi_trunc(x):
    """The REDUX key of screen.cu: the high word of a positive double, low word cleared."""
    (bits,) = struct.unpack("<Q", struct.pack("<d", x))
    return struct.unpack("<d", struct.pack("<Q", bits & 0xFFFFFFFF00000000))[0]


def record(C, pairs, P0, Q0):
    """K1: min over entries and pairs of RD(C - RU(p + q)), truncated, shifted by the counters."""
    smin = math.inf
    for p, q in pairs:
        for i, pi in enumerate(p):
            for j, qj in enumerate(q):
                v = rd_sub(C[i][j], ru_add(pi, qj))
                smin = smin if v != v else min(smin, v)  # fmin: a NaN operand is dropped
    if not smin > 0:
        return -math.inf
    return rd_add(rd_add(hi_trunc(smin), P0), Q0)


def certified(R, P, Q):
    """K0: RD(RD(record - P) - Q) > 0."""
    return rd_sub(rd_sub(R, P), Q) > 0


def exact_ok(C, pairs):
    return all(F(pi) + F(qj) < F(C[i][j]) for p, q in pairs for i, pi in enumerate(p) for j, qj in enumerate(q))


def _walk(seed):
    """One random dual walk; asserts exactness at every certified step, returns their count."""
    rng = random.Random(seed)
    rows, cols = 3, 4
    scale = rng.choice([1.0, 1e3, 3.2e4])
    C = [[scale * rng.uniform(0.5, 1.0) for _ in range(cols)] for _ in range(rows)]
    # duals just below C - margin, with margins down to the rounding level
    margin = scale * rng.choice([1e-3, 1e-8, 1e-13, 1e-15])
    cur = ([min(C[i]) * 0.5 for i in range(rows)], [0.0] * cols)
    cur = (cur[0], [min(C[i][j] - cur[0][i] for i in range(rows)) - margin for j in range(cols)])
    avg = ([x - margin * rng.random() for x in cur[0]], list(cur[1]))
    P = Q = 0.0  # one band, one cell: a single pair of counters
    R = record(C, [cur, avg], P, Q)
    step = margin * rng.choice([1e-3, 0.1, 0.5, 2.0])
    checks = 0
    for _ in range(60):
        kind = rng.random()
        new_cur = ([x + rng.uniform(-step, step) for x in cur[0]], [x + rng.uniform(-step, step) for x in cur[1]])
        new_avg = ([(a + b) / 2 for a, b in zip(avg[0], new_cur[0])], [(a + b) / 2 for a, b in zip(avg[1], new_cur[1])])
        # K2 counts the trial's drift whatever the controller decides
        D = max(max(absdiff_ru(a, b) for a, b in zip(new_cur[0], cur[0])),
                max(absdiff_ru(a, b) for a, b in zip(new_avg[0], avg[0])))
        E = max(max(absdiff_ru(a, b) for a, b in zip(new_cur[1], cur[1])),
                max(absdiff_ru(a, b) for a, b in zip(new_avg[1], avg[1])))
        P, Q = ru_add(P, D), ru_add(Q, E)
        if kind < 0.1:      # rejected trial: the duals stay
            pass
        elif kind < 0.15:   # restart: both pairs become one of this pass's two input pairs
            cand = cur if rng.random() < 0.5 else avg
            cur, avg = cand, cand
        else:               # accept
            cur, avg = new_cur, new_avg
        if certified(R, P, Q):
            checks += 1
            assert exact_ok(C, [cur, avg])
        if rng.random() < 0.2:  # K1 refreshes the record when it computes the cell
            R = record(C, [cur, avg], P, Q)
    return checks


@pytest.mark.parametrize("seed", range(40))
def test_certificate_implies_no_violation(seed):
    _walk(seed)


def test_certificates_engage():
    """The walks above are not vacuous: most steps are certified."""
    assert sum(_walk(seed) for seed in range(40)) > 40 * 60 // 4


def test_nan_and_inf_never_certify():
    """fmin drops a NaN entry from the record (as on the device), but the same
    pass's K2 turns the band's drift counter into NaN / inf, and the test fails."""
    C = [[1.0]]
    for bad in (math.nan, math.inf, -math.inf):
        R = record(C, [([bad], [0.0]), ([0.0], [0.0])], 0.0, 0.0)
        P = ru_add(0.0, absdiff_ru(bad + 0.5, bad))  # p+ - p of a non-finite dual
        assert not certified(R, P, 0.0)
        assert not certified(R, ru_add(P, 1.0), 0.0)
