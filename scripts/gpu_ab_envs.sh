# A/B of runtime switches: each argument is NAME=VAR=value[,VAR=value]; "base" is the
# default environment.  C3 bench (complete solves) twice per arm, alternating, plus a
# pass timeline per arm.  Summarise with scripts/ab_bench.py base NAME...
set -x
mkdir -p gpurun_out
names="base"
for a in "$@"; do names="$names ${a%%=*}"; done
envof() { for a in "$@"; do :; done; }
for rep in 1 2; do
  for n in $names; do
    E=""
    for a in "$@"; do [ "${a%%=*}" = "$n" ] && E=$(echo "${a#*=}" | tr ',' ' '); done
    env $E timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-variant \
      > gpurun_out/abb_${n}_$rep.json 2> gpurun_out/abb_${n}_$rep.err; echo $n $rep rc=$?
  done
done
for n in $names; do
  E=""
  for a in "$@"; do [ "${a%%=*}" = "$n" ] && E=$(echo "${a#*=}" | tr ',' ' '); done
  env $E timeout 300 python scripts/k2_trace.py 128 400 > gpurun_out/abb_${n}_trace.txt 2>&1
done
