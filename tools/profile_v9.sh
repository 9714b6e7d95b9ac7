# Round-1 v9 evidence: launch list of the bench command + full captures of the
# forward / backward rasterizers and the front stages (one launch each).
# Run on a B200:  gpurun -- bash tools/profile_v9.sh TAG
set -x
TAG=${1:-v9}
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --pool 1 --no-neurf --no-conventional --no-fast-exp --train-steps 1"
$CMD > gpurun_out/plain_$TAG.json 2> gpurun_out/plain_$TAG.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch list rc=$?"
for K in k_raster k_raster_bwd k_project k_bin_expand k_bin_scatter k_filter; do
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"${K}[<(]" -s 3 -c 1 \
      -o gpurun_out/prof_${TAG}_$K $CMD > gpurun_out/ncu_${TAG}_$K.log 2>&1
  echo "$K rc=$?"
done
ls -la gpurun_out
