"""How tight is the cell screen?  Runs a C3 solve to a few iteration counts,
takes the current iterate (X, p, q) and the average's duals (pa, qa), and
counts on the device, per 8x16 cell:
  listed      occupied (X != 0) or the screen bound fails for either dual pair
  exact       occupied or some entry violates p_i + q_j <= C_ij (either pair)
and how many listed-but-not-exact cells finer bounds would drop:
  rows        per row: p_i + max_cell q <= min_j C_ij  (8 min C per cell)
  sub4x8      four 4x8 sub-blocks, each with its own max p / max q / min C
  sub2x8      eight 2x8 sub-blocks
Usage: python scripts/screen_bound_probe.py [r=128] [iters...]"""
import ctypes
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2407_19689_b200 as pd  # noqa: E402
from paper_2407_19689_b200 import _lib  # noqa: E402
from paper_2407_19689_b200.engine import config_struct  # noqa: E402
from paper_2407_19689_b200.device import get_handle, as_device_problem  # noqa: E402

r = int(sys.argv[1]) if len(sys.argv) > 1 else 128
marks = [int(a) for a in sys.argv[2:]] or [100, 300, 600, 1000]
dp = pd.DeviceProblem.sqeuclid_grid(r, 0)
m, n = dp.m, dp.n
h = get_handle(m, n, 0)
as_device_problem(dp, 0, handle=h)
h.bind(dp)
h.set_slot(0, None, None, None)
cfg = config_struct(pd.SolverConfig(tol=1e-12, max_iters=max(marks) + 10), trace_level=0)
_lib.check(h.lib.pdot_begin(h.ptr, ctypes.byref(cfg), 0.0))
prog = _lib.Progress()
C = dp.C_t[:, :n]
B, W = 8, 16


def blk(t, bh, bw):  # (m, n) -> (m/bh, bh, n/bw, bw)
    return t.view(m // bh, bh, n // bw, bw)


def bound_fail(p, q, bh, bw, Cmin):
    pm = p.view(-1, bh).amax(1)
    qm = q.view(-1, bw).amax(1)
    return (pm[:, None] + qm[None, :]) > Cmin


DRIFT = True
cmin = {(bh, bw): blk(C, bh, bw).amin((1, 3)) for (bh, bw) in ((8, 16), (4, 8), (2, 8))}
cmin_row = C.view(m, n // W, W).amin(2)  # (m, cells)
out = []
done = 0
for mark in marks:
    while done < mark:
        _lib.check(h.lib.pdot_advance(h.ptr, 1, ctypes.byref(prog)))
        if prog.done:
            break
        done = prog.iterations
    X, p, q = h.get_slot(prog.roles[0])
    _, pa, qa = h.get_slot(prog.roles[1], want_X=False)
    Xt = torch.from_numpy(X).cuda()
    occ = blk(Xt, B, W).ne(0).any(3).any(1)
    del Xt
    duals = [(torch.from_numpy(p).cuda(), torch.from_numpy(q).cuda()),
             (torch.from_numpy(pa).cuda(), torch.from_numpy(qa).cuda())]
    listed = occ.clone()
    viol = torch.zeros_like(occ)
    rows = torch.zeros_like(occ)
    sub48 = torch.zeros_like(occ)
    sub28 = torch.zeros_like(occ)
    for pp, qq in duals:
        listed |= bound_fail(pp, qq, B, W, cmin[(8, 16)])
        for i0 in range(0, m, 2048):  # exact test in row chunks
            v = (pp[i0:i0 + 2048, None] + qq[None, :]) > C[i0:i0 + 2048]
            viol[i0 // B:(i0 + 2048) // B] |= v.view(2048 // B, B, n // W, W).any(3).any(1)
        qm = qq.view(-1, W).amax(1)
        rf = (pp[:, None] + qm[None, :]) > cmin_row  # (m, cells)
        rows |= rf.view(m // B, B, n // W).any(1)
        f48 = bound_fail(pp, qq, 4, 8, cmin[(4, 8)])  # (m/4, n/8)
        sub48 |= f48.view(m // B, 2, n // W, 2).any(3).any(1)
        f28 = bound_fail(pp, qq, 2, 8, cmin[(2, 8)])
        sub28 |= f28.view(m // B, 4, n // W, 2).any(3).any(1)
    exact = occ | viol
    loose = listed & ~exact
    rec = {"iterations": int(prog.iterations), "cells": occ.numel(), "occupied": int(occ.sum()),
           "listed": int(listed.sum()), "exact": int(exact.sum()), "listed_not_exact": int(loose.sum()),
           "kept_by_rows": int((loose & rows).sum()), "kept_by_sub4x8": int((loose & sub48).sum()),
           "kept_by_sub2x8": int((loose & sub28).sum())}
    # slack records: min over the cell of C - p_i - q_j (both pairs) taken now;
    # after k more accepted iterations a loose cell is provably inactive if
    # its record exceeds the summed per-iteration drift of the band's p and
    # the cell's q (max |change| per step)
    if DRIFT:
        def slack(pp, qq):
            s = torch.empty((m // B, n // W), dtype=torch.float64, device="cuda")
            for i0 in range(0, m, 2048):
                v = C[i0:i0 + 2048] - pp[i0:i0 + 2048, None] - qq[None, :]
                s[i0 // B:(i0 + 2048) // B] = v.view(2048 // B, B, n // W, W).amin(3).amin(1)
            return s
        s0 = [slack(pp, qq) for pp, qq in duals]
        cum = [torch.zeros(m // B, dtype=torch.float64, device="cuda"),
               torch.zeros(n // W, dtype=torch.float64, device="cuda"),
               torch.zeros(m // B, dtype=torch.float64, device="cuda"),
               torch.zeros(n // W, dtype=torch.float64, device="cuda")]
        prev = duals
        it0 = prog.iterations
        for k in range(1, 9):
            while prog.iterations < it0 + k and not prog.done:
                _lib.check(h.lib.pdot_advance(h.ptr, 1, ctypes.byref(prog)))
            if prog.done:
                break
            _, p1, q1 = h.get_slot(prog.roles[0], want_X=False)
            _, pa1, qa1 = h.get_slot(prog.roles[1], want_X=False)
            cur = [(torch.from_numpy(p1).cuda(), torch.from_numpy(q1).cuda()),
                   (torch.from_numpy(pa1).cuda(), torch.from_numpy(qa1).cuda())]
            ok = torch.ones_like(occ)
            for t, ((pp, qq), (pq0, qq0)) in enumerate(zip(cur, prev)):
                cum[2 * t] += (pp - pq0).abs().view(-1, B).amax(1)
                cum[2 * t + 1] += (qq - qq0).abs().view(-1, W).amax(1)
                ok &= (s0[t] - cum[2 * t][:, None] - cum[2 * t + 1][None, :]) > 0
            prev = cur
            if k in (1, 2, 4, 8):
                rec[f"loose_skippable_after_{k}"] = int((loose & ok).sum())
        done = prog.iterations
    print(json.dumps(rec), flush=True)
    out.append(rec)
    if prog.done:
        break
_lib.check(h.lib.pdot_finish(h.ptr, ctypes.byref(_lib.Result())))
