"""Slack certificates (K0 dropping a listed cell whose recorded slack still
exceeds the dual drift since it was recorded) against the plain cell screen
(PDOT_SREC=0): the same screened solves, bit for bit, with fewer cells visited.
The switch is read once per process, so each arm runs in its own interpreter.
Cases: the sq-Euclidean grid (many restarts), the rectangular L1 cost, the
matrix-free cost, restarts through the host-evaluated primal weight, and C2
(4096^2 to tol 1e-6: ~3.7k iterations, ~30 restarts)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import hashlib, json, sys
sys.path.insert(0, sys.argv[1])
import numpy as np
import paper_2407_19689_b200 as pd
from paper_2407_19689_b200.device import set_screening
set_screening(True)
case = sys.argv[2]
if case == "grid":
    dp, tol = pd.DeviceProblem.sqeuclid_grid(32, 3), 1e-6          # 1024^2
elif case == "rect":
    dp, tol = pd.DeviceProblem.rect_l1(1, src=(16, 32), dst=(32, 64)), 1e-5  # 512 x 2048
elif case == "c2":
    dp, tol = pd.DeviceProblem.sqeuclid_grid(64, 0), 1e-6          # C2: 4096^2, the headline's smaller sibling
elif case == "implicit":
    dp, tol = pd.DeviceProblem.sqeuclid_grid(24, 5, implicit=True), 1e-6   # 576^2, C generated in-kernel
else:  # host-evaluated primal weight: every adaptive restart pauses and resumes
    dp, tol = pd.DeviceProblem.sqeuclid_grid(32, 4), 1e-5
kw = {"host_omega": True} if case == "host_omega" else {}
(slot, h), rep = pd.solve_device(dp, pd.SolverConfig(tol=tol, deterministic=True), **kw)
X, p, q = h.get_slot(slot)
st = h.screen_stats()
hx = hashlib.sha256(np.ascontiguousarray(X).tobytes() + p.tobytes() + q.tobytes()).hexdigest()
print(json.dumps({"report": rep.to_json(), "hash": hx, "iterations": rep.iterations,
                  "restarts": rep.restarts, "active_cells": st["active_cells"], "screen_on": st["screen_on"]}))
"""


def _run(case: str, srec: str) -> dict:
    env = dict(os.environ, PDOT_SREC=srec)
    out = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT), case], env=env, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["grid", "rect", "implicit", "host_omega", "c2"])
def test_slack_certificates_bit_identical(case):
    on, off = _run(case, "1"), _run(case, "0")
    assert on["screen_on"] == 1 and off["screen_on"] == 1
    assert on["iterations"] > 50
    assert on["hash"] == off["hash"]
    assert on["report"] == off["report"]
    # the certificates drop cells the coarse bound keeps
    assert on["active_cells"] < off["active_cells"], (on["active_cells"], off["active_cells"])
    print(case, "iterations", on["iterations"], "restarts", on["restarts"], "active cells", on["active_cells"],
          "vs", off["active_cells"])
