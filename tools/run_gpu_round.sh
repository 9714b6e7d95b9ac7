#!/bin/bash
# One gpurun call: GPU tests, then the bench lines of every config.
#   gpurun -- bash tools/run_gpu_round.sh TAG [pytest-args]
TAG=${1:-cur}
shift
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf "$@" > gpurun_out/gputest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest_$TAG.log
for CFG in av2 street toy drive; do
  EXTRA=""
  [ "$CFG" != "av2" ] && EXTRA="--no-cpu-baseline --no-neurf --no-conventional --no-fast-exp --train-steps 2"
  timeout 600 python bench.py --config $CFG --steps 10 --warmup 3 $EXTRA \
      > gpurun_out/bench_${TAG}_$CFG.json 2> gpurun_out/bench_${TAG}_$CFG.err
  echo "bench $CFG rc=$?"
done
