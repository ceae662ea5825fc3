#!/bin/bash
# search parity tests + the bench's ADC section (quick)
TAG=${1:-a}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "search or query or adc or ivf or scan or config3" > gpurun_out/adc_test_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/adc_test_$TAG.log
python bench.py --no-cpu > gpurun_out/bench_adc_$TAG.json 2> gpurun_out/bench_adc_$TAG.err; echo "bench rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/bench_adc_$TAG.json').read().strip().splitlines()[-1])
a=d['adc']; print(json.dumps({k:a[k] for k in ('queries_per_s','ms_per_batch','kernel_ms_per_batch')}), a['roofline_scan']['frac'], a['roofline_lut']['frac'])
"
