"""Probe (measurement tooling, not product): how much of the m x n plan is
*active* per PDHG pass on the sq-Euclidean grid instances.

An entry (i, j) is inactive in the pass that steps from (X_t, p_t, q_t) when
X_t[i,j] == 0, the (lazy) previous average A_{t-1}[i,j] == 0, and neither the
current nor the averaged duals violate it (p_i + q_j <= C_ij and
pbar_i + qbar_j <= C_ij).  Then every output and every reduction term of that
entry is exactly zero.  The probe reruns restarted PDHG (the oracle loop, in
torch fp64 on the GPU; trajectory not bit-identical, statistics are what
matter) and reports, per pass, the active fraction at element level and for
blocks screened by a bound:

  block (I, J) must be visited iff RN(max_I p + max_J q) >= min_{I x J} C
  (same for the averaged duals) or X_t / A_{t-1} has a nonzero in it.

Usage: python scripts/active_probe.py R [seed] [tol] [max_iters]
"""
import json
import math
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2407_19689_b200 import instances as inst  # noqa: E402

r = int(sys.argv[1])
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-4
max_iters = int(sys.argv[4]) if len(sys.argv) > 4 else 100000
dev = "cuda" if torch.cuda.is_available() else "cpu"
m = n = r * r
k = torch.arange(m, device=dev, dtype=torch.float64)
a, b = torch.div(k, r, rounding_mode="floor"), k % r
C = (a[:, None] - a[None, :]) ** 2 + (b[:, None] - b[None, :]) ** 2
f_np, g_np = inst.whitenoise_marginals(r, seed)
f = torch.tensor(f_np, device=dev)
g = torch.tensor(g_np, device=dev)
fro_C = float(torch.linalg.norm(C))
marg = float(torch.linalg.norm(f) + torch.linalg.norm(g))

BS = [(8, 8), (16, 16), (8, 64), (16, 64), (32, 32), (64, 64), (2, 512), (128, 512)]
BS = [bb for bb in BS if bb[1] <= n]
minC = {bb: C.reshape(m // bb[0], bb[0], n // bb[1], bb[1]).amin(dim=(1, 3)) for bb in BS}
# row-level bound: min over a column block for each row
RB = [bn for bn in (64, 512) if bn <= n]
minCrow = {bn: C.reshape(m, n // bn, bn).amin(dim=2) for bn in RB}


def bmax(v, s):
    return v.reshape(-1, s).amax(dim=1)


def bany(X, bm, bn):
    return (X.reshape(m // bm, bm, n // bn, bn) != 0).any(dim=3).any(dim=1)


stats = {str(bb): [] for bb in BS}
stats.update({f"row{bn}": [] for bn in RB})
stats["elem"] = []
stats["x_density"] = []
stats["a_density"] = []


def record(X, p, q, A_prev, pb, qb):
    nzx = X != 0
    nza = A_prev != 0
    pq = p[:, None] + q[None, :]
    el = nzx | nza | (pq > C) | ((pb[:, None] + qb[None, :]) > C)
    stats["elem"].append(float(el.double().mean()))
    stats["x_density"].append(float(nzx.double().mean()))
    stats["a_density"].append(float(nza.double().mean()))
    for bb in BS:
        bm, bn = bb
        mc = minC[bb]
        act = ((bmax(p, bm)[:, None] + bmax(q, bn)[None, :]) >= mc) | \
              ((bmax(pb, bm)[:, None] + bmax(qb, bn)[None, :]) >= mc) | bany(X, bm, bn) | bany(A_prev, bm, bn)
        stats[str(bb)].append(float(act.double().mean()))
    for bn in RB:
        mc = minCrow[bn]
        act = ((p[:, None] + bmax(q, bn)[None, :]) >= mc) | ((pb[:, None] + bmax(qb, bn)[None, :]) >= mc) | \
              (X.reshape(m, n // bn, bn) != 0).any(dim=2) | (A_prev.reshape(m, n // bn, bn) != 0).any(dim=2)
        stats[f"row{bn}"].append(float(act.double().mean()))


def step(X, p, q, tau, sigma):
    Xn = torch.clamp_min(X - tau * (C - (p[:, None] + q[None, :])), 0.0)
    E = 2.0 * Xn - X
    return Xn, p + sigma * (f - E.sum(1)), q + sigma * (g - E.sum(0))


def kkt(X, p, q):
    pr, pc = X.sum(1) - f, X.sum(0) - g
    viol = torch.clamp_min(p[:, None] + q[None, :] - C, 0.0)
    pobj = float((C * X).sum())
    dobj = float(f @ p + g @ q)
    gap = pobj - dobj
    psq = float(pr @ pr + pc @ pc)
    dsq = float((viol * viol).sum())
    return math.sqrt(psq) / (1 + marg) + math.sqrt(dsq) / (1 + fro_C) + abs(gap) / (1 + abs(pobj) + abs(dobj))


X = torch.zeros(m, n, device=dev, dtype=torch.float64)
p = torch.zeros(m, device=dev, dtype=torch.float64)
q = torch.zeros(n, device=dev, dtype=torch.float64)
eta, omega = 1.0 / (2.0 * math.sqrt(m + n)), 1.0
z = kkt(X, p, q)
anchor = (X.clone(), p.clone(), q.clone())
avg = (X.clone(), p.clone(), q.clone())
A_prev = X.clone()
prev, total, inner, restarts, passes = z, 0, 0, 0, 0
t0 = time.time()
while total < max_iters:
    pb, qb = avg[1], avg[2]
    for _ in range(80):
        record(X, p, q, A_prev, pb, qb)
        passes += 1
        Xn, pn, qn = step(X, p, q, eta / omega, eta * omega)
        dX, dp, dq = Xn - X, pn - p, qn - q
        num = omega * float((dX * dX).sum()) + float(dp @ dp + dq @ dq) / omega
        den = 2.0 * abs(float(dp @ dX.sum(1) + dq @ dX.sum(0)))
        bnd = math.inf if den <= 1e-10 else num / den
        if eta <= bnd:
            if math.isfinite(bnd):
                eta = min(1.05 * eta, bnd)
            break
        eta *= 0.5
    A_prev = avg[0]
    X, p, q = Xn, pn, qn
    total += 1
    inner += 1
    avg = (avg[0] + (X - avg[0]) / inner, avg[1] + (p - avg[1]) / inner, avg[2] + (q - avg[2]) / inner)
    kc, ka = kkt(X, p, q), kkt(*avg)
    cand, ck = ((X, p, q), kc) if kc < ka else (avg, ka)
    if ck <= tol:
        break
    fire = ck <= 0.1 * z or (ck <= 0.9 * z and ck > prev) or inner >= 0.36 * total
    if fire:
        dXn = float(torch.linalg.norm(cand[0] - anchor[0]))
        dpq = math.sqrt(float(((cand[1] - anchor[1]) ** 2).sum() + ((cand[2] - anchor[2]) ** 2).sum()))
        if dXn > 1e-10 and dpq > 1e-10:
            omega = math.exp(0.5 * math.log(dpq / dXn) + 0.5 * math.log(omega))
        X, p, q = (t.clone() for t in cand)
        anchor = (X.clone(), p.clone(), q.clone())
        avg = (X.clone(), p.clone(), q.clone())
        A_prev = X.clone()
        z, prev, inner = ck, ck, 0
        restarts += 1
    else:
        prev = ck
out = {"r": r, "seed": seed, "tol": tol, "iterations": total, "restarts": restarts, "passes": passes,
       "seconds": time.time() - t0, "final_kkt": ck}
for key, v in stats.items():
    t = torch.tensor(v, dtype=torch.float64)
    out[key] = {"mean": float(t.mean()), "max": float(t.max()), "last": float(t[-1]),
                "p90": float(t.quantile(0.9))}
print(json.dumps(out))
