#!/bin/bash
# r2e evidence in one call: bench line + encode ncu capture + launch lists
# (gpu_bench_prof.sh), ncu --set full of the recon SSE kernel (D=128 M=16 and
# D=96 M=12) and of the k-means update kernels (warm cache, eager fit).
TAG=${1:-r2e}
mkdir -p gpurun_out
bash tools/gpu_bench_prof.sh $TAG
for a in "128 16" "96 12"; do
  set -- $a
  ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:recon_sse \
      -o gpurun_out/sse_${TAG}_d$1m$2 -f python tools/sse_bench.py --d $1 --m $2 --ncu > /dev/null 2>&1
  echo "ncu sse d$1 m$2 rc=$?"
done
PQG_KM_GRAPH=0 ncu --set full --cache-control none --clock-control none --import-source on \
    -k regex:"mean_pieces|scatter_kernel|mean_replay|pieces_setup|hist_kernel|mean_finalize|partial_sum|reseed" \
    --launch-skip 40 --launch-count 8 -o gpurun_out/km_upd_$TAG -f python tools/kmeans_breakdown.py --no-coarse \
    > /dev/null 2>&1
echo "ncu kmeans rc=$?"
