# Evidence for profiles/: the launch list of the bench command, then full
# captures (ncu --set full) of one launch each of the rasterizers and the front
# stages.  Run on a B200:  gpurun -- bash tools/profile_round.sh TAG
# then here:  python tools/ncu_summary.py profiles/r01_ncu_full_TAG.json gpurun_out/prof_TAG_*.ncu-rep
#             python tools/ncu_traffic.py profiles/r01_ncu_full_TAG.json av2
set -x
TAG=${1:-cur}
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --pool 1 --no-neurf --no-conventional --no-fast-exp --train-steps 1"
$CMD > gpurun_out/plain_$TAG.json 2> gpurun_out/plain_$TAG.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch list rc=$?"
# kernel:launches to skip (the training kernels run once per train step only)
for KS in k_raster:3 k_raster_bwd:1 k_project_bwd:1 k_project:3 k_bin_expand:3 k_bin_scatter:3 k_filter:3 k_onesweep:20; do
  K=${KS%%:*}; S=${KS##*:}
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:"${K}[<(]" -s $S -c 1 -o gpurun_out/prof_${TAG}_$K $CMD > gpurun_out/ncu_${TAG}_$K.log 2>&1
  echo "$K rc=$?"
done
ls -la gpurun_out
