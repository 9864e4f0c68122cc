"""Per-shard latency model of a row-sharded screened pass from an ncu launch list
of scripts/shard_probe.py (gpu__time_duration per launch, serialised, cold-ish):

    python scripts/shard_model.py R launches.csv

Prints, per phase, the mean over passes of the slowest shard's kernel time:
phase 0 = K0 + K1 + K1b + K2a (local rows), phase 1 = K2b (combine of the 8
groups + controller, identical work on every rank)."""
import csv
import json
import sys
from collections import defaultdict


def main(R, path):
    rows = []
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v = v * {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
        name = r["Kernel Name"]
        k = next((s for s in ("screen_kernel", "unit_kernel", "tile_kernel", "finalize_kernel") if s in name), None)
        if k:
            rows.append((k, v))
    per = 5 * R  # launches per pass
    npass = len(rows) // per
    acc = defaultdict(list)
    for p in range(npass):
        chunk = rows[p * per:(p + 1) * per]
        ph0 = [sum(v for _, v in chunk[4 * r:4 * r + 4]) for r in range(R)]
        k1 = [chunk[4 * r + 1][1] for r in range(R)]
        k0 = [chunk[4 * r][1] for r in range(R)]
        k1b = [chunk[4 * r + 2][1] for r in range(R)]
        k2a = [chunk[4 * r + 3][1] for r in range(R)]
        k2b = [v for _, v in chunk[4 * R:]]
        for key, vals in (("phase0_max", ph0), ("k0_max", k0), ("k1_max", k1), ("k1b_max", k1b),
                          ("k2a_max", k2a), ("k2b_max", k2b)):
            acc[key].append(max(vals))
    out = {k: sum(v) / len(v) for k, v in acc.items()}
    out.update(R=R, passes=npass, unit="us")
    print(json.dumps(out))


if __name__ == "__main__":
    main(int(sys.argv[1]), sys.argv[2])
