# ncu full captures of the backward kernels (config 5).  gpurun -- bash tools/profile_bwd.sh TAG
set -x
TAG=${1:-bwd}
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --pool 1 --train-steps 1"
$CMD > gpurun_out/plain_$TAG.json 2> gpurun_out/plain_$TAG.err && \
for K in k_raster_bwd k_project_bwd k_mse; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
      -o gpurun_out/prof_${TAG}_$K $CMD > gpurun_out/ncu_${TAG}_$K.log 2>&1
  echo "$K rc=$?"
done
