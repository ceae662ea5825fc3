set -x
for c in 0 4 5 6 8; do
  if [ $c = 0 ]; then unset PQG_UMMA_CTAS; else export PQG_UMMA_CTAS=$c; fi
  echo "CTAS=$c"
  timeout 300 python tools/encode_bench.py --points 16x64,32x64,16x256,32x256,4x64,8x64 --reps 10 2>&1 | grep '^{'
done
