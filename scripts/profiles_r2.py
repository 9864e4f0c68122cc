"""Copy the round-2 final measurement set (scripts/gpu_measure_r2.sh -> gpurun_out/f_*)
into profiles/: bench lines, -m gpu suite log, ncu launch list, --set full summaries,
K1 warm DRAM traffic, pass timeline and screen trace.  Usage: python scripts/profiles_r2.py"""
import csv
import json
import shutil
import sys

sys.path.insert(0, "scripts")
import summarize_ncu as S  # noqa: E402

for c in ("c3", "c1", "c2", "c4", "ref"):
    line = open(f"gpurun_out/f_{c}.json").read().strip().splitlines()[-1]
    open(f"profiles/r02_bench_{c}.json", "w").write(line + "\n")
L = S.launches("gpurun_out/f_launches.csv")
json.dump({"how": "ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv python bench.py --steps 2 "
                  "--warmup 3 --no-e2e --no-variant --no-cpu (final round-2 build; every step a complete C3 solve; "
                  "serialised and cold-ish under ncu: compare shares, not absolutes)", "kernels": L},
          open("profiles/r02_launches_c3.json", "w"), indent=1)
full = {"how": "ncu --set full --clock-control none --import-source on -k regex:<kernel> --launch-skip 300 "
               "--launch-count 1 python scripts/prof_solve.py 128 500 (mid-solve C3 pass of the final round-2 build; "
               "kernel replayed in isolation: cold L2, warm instruction cache)"}
for k in ("unit_kernel", "screen_kernel", "tile_kernel", "finalize_kernel"):
    full[k] = S.full(f"gpurun_out/f_full_{k}.ncu-rep")
json.dump(full, open("profiles/r02_screened_kernels_ncu.json", "w"), indent=1)
rows = list(csv.reader(open("gpurun_out/f_k1_dram.csv")))
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
alg = json.loads(open("gpurun_out/f_k1_alg.json").read().strip().splitlines()[-1])
t = json.load(open("profiles/screened_kernel_traffic.json"))
t.update({"launches": n, "dram_read_bytes": rd, "dram_write_bytes": wr, "algorithmic_bytes": alg["k1_bytes"],
          "dram_to_algorithmic": (rd + wr) / alg["k1_bytes"],
          "source": "gpurun_out/f_k1_dram.csv, gpurun_out/f_k1_alg.json (round 2, final build)"})
json.dump(t, open("profiles/screened_kernel_traffic.json", "w"), indent=1)
shutil.copy("gpurun_out/f_k2trace.txt", "profiles/r02_pass_timeline.txt")
shutil.copy("gpurun_out/f_screen_trace.txt", "profiles/r02_screen_trace_c3.txt")
with open("profiles/r02_gpu_suite.log", "w") as fo:
    fo.write(open("gpurun_out/f_suite.log").read()[-3000:])
    fo.write("\n--- smoke()\n" + open("gpurun_out/f_smoke.log").read()[-1000:])
for c in ("c3", "c1", "c2", "c4", "ref"):
    d = json.loads(open(f"profiles/r02_bench_{c}.json").read())
    tt = d.get("time_to_tol") or {}
    print(c, round(d["value"], 3), "tol", tt.get("device_s_mean"), tt.get("iterations"), "e2e",
          round((d.get("e2e") or {}).get("value", 0), 1), "roof", (d.get("roofline") or {}).get("frac"), d.get("clocks"))
print("K1 dram/alg", t["dram_to_algorithmic"])
for k in L[:6]:
    print(k["kernel"], k["launches"], round(k["mean_us"], 2), round(k["share"], 3))
print(open("profiles/r02_pass_timeline.txt").read().splitlines()[0])
