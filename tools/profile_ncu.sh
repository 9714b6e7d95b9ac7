# ncu evidence for profiles/: the launch list of the bench command, then full
# captures of the top kernels (one launch each, after warm-up).
# Run on a B200:  gpurun -- bash tools/profile_ncu.sh [tag]
set -x
TAG=${1:-cur}
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --pool 1"
$CMD > gpurun_out/plain_$TAG.json 2> gpurun_out/plain_$TAG.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch list rc=$?"
for K in k_raster k_project k_bin_expand k_bin_scatter k_permute k_filter k_raster_bwd k_project_bwd k_neurf k_to_world; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
      -o gpurun_out/prof_${TAG}_$K $CMD > gpurun_out/ncu_${TAG}_$K.log 2>&1
  echo "$K rc=$?"
done
ncu --set full --clock-control none --import-source on -k regex:k_onesweep -s 20 -c 1 \
    -o gpurun_out/prof_${TAG}_onesweep $CMD > gpurun_out/ncu_${TAG}_onesweep.log 2>&1
echo "onesweep rc=$?"
ls -la gpurun_out
