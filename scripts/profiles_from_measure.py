"""Copy one gpu_measure_all.sh run (gpurun_out/m_*) into profiles/ under a version tag:
bench lines, ncu launch list, --set full summaries, K1 warm DRAM traffic, pass timeline,
screen trace.  Usage: python scripts/profiles_from_measure.py v12"""
import csv
import json
import shutil
import sys

sys.path.insert(0, "scripts")
import summarize_ncu as S  # noqa: E402

V = sys.argv[1]
for c in ("c3", "c1", "c2", "c4", "ref"):
    line = open(f"gpurun_out/m_{c}.json").read().strip().splitlines()[-1]
    open(f"profiles/r01_bench_{c}_{V}.json", "w").write(line + "\n")
L = S.launches("gpurun_out/m_launches.csv")
json.dump({"how": "ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 python bench.py --steps 120 "
                  "--warmup 5 --no-tol --no-e2e --no-variant --no-cpu (C3, screened passes; per-launch times are "
                  "serialised and cold-cache under ncu: compare shares, not absolutes)", "kernels": L},
          open(f"profiles/r01_launches_screened_{V}.json", "w"), indent=1)
full = {"how": "ncu --set full --clock-control none --import-source on -k regex:<kernel> --launch-skip 90 "
               "--launch-count 1, same bench command (cold cache)"}
for k in ("unit_kernel", "screen_kernel", "tile_kernel", "finalize_kernel"):
    full[k] = S.full(f"gpurun_out/m_full_{k}.ncu-rep")
json.dump(full, open(f"profiles/r01_screened_kernels_ncu_{V}.json", "w"), indent=1)
rows = list(csv.reader(open("gpurun_out/m_k1_dram.csv")))
hi = next(i for i, r in enumerate(rows) if "Metric Name" in r)
h = rows[hi]
mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd = wr = 0.0
n = 0
for r in rows[hi + 1:]:
    if r[mi] == "dram__bytes_read.sum":
        rd += float(r[vi].replace(",", "")) * scale[r[ui]]
        n += 1
    elif r[mi] == "dram__bytes_write.sum":
        wr += float(r[vi].replace(",", "")) * scale[r[ui]]
alg = json.load(open("gpurun_out/m_k1_alg.json"))
t = json.load(open("profiles/screened_kernel_traffic.json"))
t.update({"launches": n, "dram_read_bytes": rd, "dram_write_bytes": wr, "algorithmic_bytes": alg["k1_bytes"],
          "dram_to_algorithmic": (rd + wr) / alg["k1_bytes"],
          "source": f"gpurun_out/m_k1_dram.csv, gpurun_out/m_k1_alg.json (round 1, {V})"})
json.dump(t, open("profiles/screened_kernel_traffic.json", "w"), indent=1)
shutil.copy("gpurun_out/m_k2trace.txt", f"profiles/r01_pass_timeline_{V}.txt")
shutil.copy("gpurun_out/m_screen_trace.txt", f"profiles/r01_screen_trace_c3_{V}.txt")
for c in ("c3", "c1", "c2", "c4", "ref"):
    d = json.loads(open(f"profiles/r01_bench_{c}_{V}.json").read())
    tt = d.get("time_to_tol") or {}
    print(c, round(d["value"], 3), "tol", tt.get("seconds"), tt.get("iterations"), "e2e",
          round((d.get("e2e") or {}).get("value", 0), 1), "roof", (d.get("roofline") or {}).get("frac"), d.get("clocks"))
print("K1 dram/alg", t["dram_to_algorithmic"])
for k in L[:6]:
    print(k["kernel"], k["launches"], round(k["mean_us"], 2), round(k["share"], 3))
print(open(f"profiles/r01_pass_timeline_{V}.txt").read().splitlines()[0])
