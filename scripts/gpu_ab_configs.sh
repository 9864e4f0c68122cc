# A/B of a prebuilt library variant (lib/variants/$1.so) against the in-tree build on
# several configs ($2.., e.g. c3 c4): complete-solve bench lines, alternating, twice
set -x
V=$1; shift
for rep in 1 2; do
  for c in "$@"; do
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-variant > gpurun_out/abc_base_${c}_$rep.json 2>/dev/null
    PDOT_LIB_PATH=$PWD/paper_2407_19689_b200/lib/variants/$V.so timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-variant > gpurun_out/abc_${V}_${c}_$rep.json 2>/dev/null
  done
done
python - "$V" "$@" <<'PY'
import json, sys
V = sys.argv[1]
for c in sys.argv[2:]:
    for arm in ("base", V):
        vals = []
        for rep in (1, 2):
            try:
                d = json.loads(open(f"gpurun_out/abc_{arm}_{c}_{rep}.json").read().strip().splitlines()[-1])
                vals.append((round(d["value"]), round(d["screening"]["pass_us_mean"], 1) if d.get("screening") else None))
            except Exception as e:
                vals.append(("missing", str(e)[:30]))
        print(c, arm, vals)
PY
