"""Summarise ncu outputs into profiles/: a launch-list share table and the
key metrics of one --set full capture (run here, no GPU needed)."""
import collections
import csv
import json
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        name = r[ki].split("(")[0].split("::")[-1]
        v = float(r[vi].replace(",", ""))
        v = v * {"ms": 1e3, "us": 1.0, "ns": 1e-3, "s": 1e6}.get(r[ui], 1.0)
        agg[name].append(v)
    tot = sum(sum(v) for v in agg.values())
    return [{"kernel": k, "launches": len(v), "mean_us": sum(v) / len(v), "total_ms": sum(v) / 1e3,
             "share": sum(v) / tot} for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))]


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u, v = r[0], r[1], r[2]
    d = {}
    for i, n in enumerate(h):
        if n in WANT:
            d[n] = {"value": v[i], "unit": u[i]}
    stalls = []
    for i, n in enumerate(h):
        if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(v[i]), n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    d["top_stalls_per_issue"] = [{"reason": s, "ratio": x} for x, s in sorted(stalls, reverse=True)[:6]]
    return d


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(json.dumps(launches(path) if kind == "launches" else full(path), indent=1))
