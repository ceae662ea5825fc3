#!/bin/bash
# full GPU test suite + the encode microbench over the configs[1] sweep
mkdir -p gpurun_out
TAG=${1:-c}
python -m pytest tests -m gpu -x -q > gpurun_out/gputest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gputest_$TAG.log
python tools/encode_bench.py --points 4x16,8x16,16x16,32x16,4x64,8x64,16x64,32x64,4x256,8x256,16x256,32x256 > gpurun_out/encbench_$TAG.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/encbench_$TAG.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print(d['M'], d['Ks'], round(d['ms'],4), round(d['G_vec_s'],3), d['exact'], {k: round(v,4) for k,v in d['kernels_ms'].items()})
"
