# Per-shard latency model of the row-sharded screened pass at C3:
# R virtual shards on one GPU (no kernel waits on another), ncu launch durations of
# 40 mid-solve passes (after 300 warm-up passes), parsed by scripts/shard_model.py.
set -x
mkdir -p gpurun_out
python scripts/shard_probe.py 2 20 || exit 1
for R in 2 4 8; do
  N=$((5 * R))
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"screen_kernel|unit_kernel|tile_kernel|finalize_kernel" \
    --launch-skip $((300 * N)) --launch-count $((40 * N)) --csv --log-file gpurun_out/shard_R$R.csv \
    python scripts/shard_probe.py $R 340 > gpurun_out/shard_R$R.out 2>&1
  echo "R=$R rc=$?"
  python scripts/shard_model.py $R gpurun_out/shard_R$R.csv
done
# the fused single-GPU pass, same window, for reference
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"screen_kernel|unit_kernel|tile_kernel|finalize_kernel" --launch-skip 1200 --launch-count 160 \
  --csv --log-file gpurun_out/shard_R1.csv python scripts/prof_solve.py 128 340 > /dev/null 2>&1
echo "R=1 rc=$?"
