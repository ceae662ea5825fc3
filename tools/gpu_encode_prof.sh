#!/bin/bash
# encode microbench over the configs[1] sweep points, then ncu --set full of
# the encode kernels at the points named in $PROF (default 32x16,32x64).
TAG=${1:-enc}
mkdir -p gpurun_out
python tools/encode_bench.py --points ${POINTS:-4x16,8x16,16x16,32x16,4x64,8x64,16x64,32x64,16x256,32x256} \
    > gpurun_out/encbench_$TAG.jsonl 2> gpurun_out/encbench_$TAG.err
echo "encode_bench rc=$?"; cat gpurun_out/encbench_$TAG.jsonl
if [ -z "$SKIP_NCU" ]; then
  for p in ${PROF:-32x16 32x64}; do
    ncu --set full --import-source on --clock-control none --profile-from-start off \
        -o gpurun_out/enc_${TAG}_$p -f python tools/encode_bench.py --points $p --ncu > gpurun_out/ncu_enc_${TAG}_$p.log 2>&1
    echo "ncu $p rc=$?"
  done
fi
