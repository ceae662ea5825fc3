#!/bin/bash
# sharded-fit GPU checks: the threaded world 1-4 tests (both replay protocols)
# and configs[4] on one 12.5M-row shard with the exchange forced, chain vs gather
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "kmshard or dist" > gpurun_out/shard_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/shard_tests.log
for r in chain gather; do
  python tools/cfg5.py --rows-per-rank 12500000 --force-exchange --replay $r > gpurun_out/cfg5_fx_$r.json 2> gpurun_out/cfg5_fx_$r.err
  echo "cfg5 $r rc=$?"; tail -c 900 gpurun_out/cfg5_fx_$r.json; echo
done
