#!/bin/bash
# quick loop: a subset of GPU parity tests ($TESTK), the encode microbench
# ($POINTS) and optional extra commands ($EXTRA)
mkdir -p gpurun_out
TAG=${1:-q}
python -m pytest tests -m gpu -x -q ${TESTK:+-k "$TESTK"} > gpurun_out/quick_$TAG.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/quick_$TAG.log
if [ -n "$POINTS" ]; then
  python tools/encode_bench.py --points $POINTS > gpurun_out/encbench_$TAG.jsonl 2> gpurun_out/encbench_$TAG.err
  echo "encode_bench rc=$?"; cat gpurun_out/encbench_$TAG.jsonl; tail -3 gpurun_out/encbench_$TAG.err
fi
if [ -n "$EXTRA" ]; then bash -c "$EXTRA"; fi
