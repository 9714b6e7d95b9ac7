# ncu evidence for profiles/: launch list of the bench command + full captures of the top kernels.
# Run on a B200 via: gpurun -- bash tools/profile_ncu.sh
set -x
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --pool 1"
$CMD > gpurun_out/plain.json 2> gpurun_out/plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
for K in k_raster k_project k_emit k_filter; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_$K $CMD > gpurun_out/ncu_$K.log 2>&1
  echo "$K rc=$?"
done
ncu --set full --clock-control none --import-source on -k regex:k_onesweep -s 14 -c 2 -o gpurun_out/prof_onesweep $CMD > gpurun_out/ncu_onesweep.log 2>&1
echo "onesweep rc=$?"
ls -la gpurun_out
