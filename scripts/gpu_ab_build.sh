# A/B of library variants built on the box: each argument is NAME=FLAGS (nvcc -D...);
# "base" is the in-tree library.  Bench C3 (complete solves) twice per arm, alternating,
# plus a K2 pass timeline per arm.  Summarise with scripts/ab_bench.py.
set -x
mkdir -p gpurun_out paper_2407_19689_b200/lib/variants
names="base"
for a in "$@"; do
  n=${a%%=*}
  if [ "$n" != "$a" ]; then  # NAME=FLAGS: build it here; a bare NAME is a prebuilt lib/variants/NAME.so
    f=${a#*=}
    PDOT_NVCC_EXTRA="$f" PDOT_BUILD_OUT=$PWD/paper_2407_19689_b200/lib/variants/$n.so \
      python -c "from paper_2407_19689_b200.build import build_library; build_library(force=True)" || exit 1
  fi
  names="$names $n"
done
for rep in 1 2; do
  for n in $names; do
    L=""; [ "$n" != base ] && L=$PWD/paper_2407_19689_b200/lib/variants/$n.so
    PDOT_LIB_PATH=$L timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-variant \
      > gpurun_out/abb_${n}_$rep.json 2> gpurun_out/abb_${n}_$rep.err; echo $n $rep rc=$?
  done
done
for n in $names; do
  L=""; [ "$n" != base ] && L=$PWD/paper_2407_19689_b200/lib/variants/$n.so
  PDOT_LIB_PATH=$L timeout 300 python scripts/k2_trace.py 128 400 > gpurun_out/abb_${n}_trace.txt 2>&1
done
