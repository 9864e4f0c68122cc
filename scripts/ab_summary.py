"""Summarise gpurun_out/ab_<variant>_{c3,c2}.json (scripts/gpu_ab_env.sh: base / var;
scripts/gpu_ab_libs.sh: one name per library variant)."""
import json
import sys

names = sys.argv[1:] or ["base", "var"]
for c in ("c3", "c2"):
    for arm in names:
        try:
            d = json.loads(open(f"gpurun_out/ab_{arm}_{c}.json").read().strip().splitlines()[-1])
        except Exception as e:  # noqa: BLE001
            print(c, arm, "missing", e)
            continue
        t = d.get("time_to_tol") or {}
        s = d.get("screening") or {}
        print(c, arm, round(d["value"]), "tol", round(t.get("seconds", 0), 4), t.get("iterations"),
              "e2e", round(d["e2e"]["value"]), "k1", round(s.get("k1_us", 0), 1), "k2", round(s.get("k2_us_to_last_block", 0), 1))
for arm in names:
    try:
        print(arm, open(f"gpurun_out/ab_{arm}_trace.txt").read().splitlines()[0])
    except Exception:  # noqa: BLE001
        pass
