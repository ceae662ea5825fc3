#!/bin/bash
# One gpurun call: GPU tests, the default bench line, and the ncu launch list
# of the same bench (taken after the plain run exited 0).  Outputs land in
# gpurun_out/ (merged back by gpurun).  Usage: bash tools/gpu_round.sh [tag]
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
if [ -z "$SKIP_TESTS" ]; then
  python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/gputest_$TAG.log 2>&1
  echo "pytest rc=$?" | tee -a gpurun_out/gputest_$TAG.log
  tail -3 gpurun_out/gputest_$TAG.log
fi
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
rc=$?; echo "bench rc=$rc"; cat gpurun_out/bench_$TAG.json | head -c 600; echo
if [ $rc -eq 0 ] && [ -z "$SKIP_NCU" ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
      --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 10 --warmup 3 --no-cpu --profile-region ${REGION:-encode} \
      > gpurun_out/ncu_bench_$TAG.log 2>&1
  echo "ncu rc=$?"
fi
