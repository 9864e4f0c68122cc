"""Summarise scripts/gpu_ab_build.sh runs: python scripts/ab_bench.py base var1 ..."""
import json
import sys

for n in sys.argv[1:]:
    vals = []
    for rep in (1, 2):
        try:
            d = json.loads(open(f"gpurun_out/abb_{n}_{rep}.json").read().strip().splitlines()[-1])
            s = d["screening"]
            vals.append((round(d["value"]), round(d["ms_per_step"], 2), round(s["k1_us"], 1),
                         round(s["k2_us_to_last_block"], 1), round(s["k2_controller_us"], 1),
                         round(s["pass_us_mean"], 1), d["time_to_tol"]["iterations"]))
        except Exception as e:  # noqa: BLE001
            vals.append(("missing", str(e)[:40]))
    print(n, "iter/s, ms/solve, K1 us, K2 us, ctl us, pass us, iterations:", vals)
    try:
        print("   ", open(f"gpurun_out/abb_{n}_trace.txt").read().splitlines()[0])
        print("   ", open(f"gpurun_out/abb_{n}_trace.txt").read().splitlines()[-1])
    except Exception:  # noqa: BLE001
        pass
