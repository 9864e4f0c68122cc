"""K2 launched as a programmatic dependent of K1b (the default) against a plain
launch (PDOT_PDL_K2=0): the same screened solve, bit for bit.  The switch is
read once per process, so each arm runs in its own interpreter."""

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
dp = pd.DeviceProblem.sqeuclid_grid(32, 3)  # 1024^2, screened passes forced
it, rep = pd.solve(dp, pd.SolverConfig(tol=1e-6, deterministic=True))
h = hashlib.sha256(np.ascontiguousarray(it.X).tobytes() + it.p.tobytes() + it.q.tobytes()).hexdigest()
print(json.dumps({"report": rep.to_json(), "hash": h, "iterations": rep.iterations}))
"""


def _run(pdl: str) -> dict:
    env = dict(os.environ, PDOT_PDL_K2=pdl)
    out = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT)], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
def test_pdl_k2_bit_identical():
    a, b = _run("1"), _run("0")
    assert a["iterations"] > 50
    assert a["hash"] == b["hash"]
    assert a["report"] == b["report"]
