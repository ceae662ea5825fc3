#!/bin/bash
# bench line + ncu evidence of the headline encode: full capture of the screen
# kernel (prof_enc_<tag>) and the launch list of bench.py's timed encode region
TAG=${1:-r2}
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"umma_screen|row_screen|narrow" \
    -o gpurun_out/prof_enc_$TAG -f python tools/encode_bench.py --points 8x256 --ncu > gpurun_out/ncu_enc_$TAG.log 2>&1
echo "ncu encode rc=$?"
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_enc_$TAG.csv python bench.py --steps 10 --warmup 3 --no-cpu --quick --profile-region encode \
    > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_adc_$TAG.csv python bench.py --steps 6 --warmup 3 --no-cpu --profile-region adc \
    > gpurun_out/ncu_launch_adc_$TAG.log 2>&1; echo "ncu adc launches rc=$?"
