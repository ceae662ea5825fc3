#!/bin/bash
# recon SSE kernel sweep (D, M) with the default path and PQG_SSE_BULK=0
for a in "--d 128 --m 16" "--d 96 --m 12" "--d 128 --m 32" "--d 128 --m 8"; do
  python tools/sse_bench.py $a | tail -1
  PQG_SSE_BULK=0 python tools/sse_bench.py $a | tail -1 | sed 's/^/bulk0 /'
done
