#!/bin/bash
# A/B (alternating): single-view launches with supertile rows issued centre-out (MFA_CENTER_OUT=1) vs raster order
for f in ${CO_FLAGS:-"-DMFA_CENTER_OUT=1" "" "-DMFA_CENTER_OUT=1" ""}; do
  echo "=== flags: $f"
  MFA_EXTRA_NVCC_FLAGS="${f#none}" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  python tools/img_hash.py 3
  MFA_BENCH_RUNS=2:0,3:0,4:0 python bench.py --all-configs --steps 3 --warmup 3 2> gpurun_out/co.err | python -c "
import json,sys
for l in sys.stdin:
    x=json.loads(l); print(x['config']['workload'][:12], round(x['value']/1e9,2), 'G/s  launch_ms', round(x['roofline']['launch_ms'],4))"
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
