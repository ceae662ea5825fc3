#!/bin/bash
# configs[3] on one GPU and one GPU's shard of configs[4] (tools/cfg4.py, tools/cfg5_shard.py)
TAG=${1:-r2}
mkdir -p gpurun_out
python tools/cfg4.py > gpurun_out/cfg4_$TAG.json 2> gpurun_out/cfg4_$TAG.err; echo "cfg4 rc=$?"; tail -c 600 gpurun_out/cfg4_$TAG.json
python tools/cfg5_shard.py > gpurun_out/cfg5_$TAG.json 2> gpurun_out/cfg5_$TAG.err; echo "cfg5 rc=$?"; tail -c 900 gpurun_out/cfg5_$TAG.json
