"""Summarise gpurun_out/ab_{base,var}_*.json (scripts/gpu_ab_env.sh)."""
import json
for c in ("c3", "c2"):
    for arm in ("base", "var"):
        try:
            d = json.loads(open(f"gpurun_out/ab_{arm}_{c}.json").read().strip().splitlines()[-1])
        except Exception as e:  # noqa: BLE001
            print(c, arm, "missing", e)
            continue
        t = d.get("time_to_tol") or {}
        s = d.get("screening") or {}
        print(c, arm, round(d["value"]), "tol", round(t.get("seconds", 0), 4), t.get("iterations"),
              "e2e", round(d["e2e"]["value"]), "k1", round(s.get("k1_us", 0), 1), "k2", round(s.get("k2_us_to_last_block", 0), 1))
print(open("gpurun_out/ab_var_trace.txt").read().splitlines()[0])
