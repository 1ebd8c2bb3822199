#!/bin/bash
# NEXT-1 transparent-block skip (shading = 3): parity (bit-identical to shading = 1) and throughput
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "skip_transparent or subset or both_layouts" 2>&1 | tail -2
for c in c5 c2; do
  for v in "" "--skip-transparent-blocks"; do
    timeout 900 python bench.py --workload $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-eval $v > gpurun_out/sb.json 2> gpurun_out/sb.err
    python -c "
import json; r=json.load(open('gpurun_out/sb.json')); print('$c', '$v', round(r['value']/1e9,2), 'G samples/s', round(r['ms_per_step'],3), 'ms', round(r['frames_per_s'],1), 'fps')" || tail -3 gpurun_out/sb.err
  done
done
