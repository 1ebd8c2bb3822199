#!/bin/bash
# quick perf sweep: device-timed render throughput for C3, C4, C5 (no e2e / cpu baseline)
for c in ${@:-c3 c4 c5}; do
  timeout 600 python bench.py --workload $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-eval $QB_ARGS > gpurun_out/qb_$c.json 2> gpurun_out/qb_$c.err
  python - "$c" <<'PY'
import json,sys
c=sys.argv[1]
try:
    r=json.load(open(f"gpurun_out/qb_{c}.json"))
    print(f"{c}: {r['value']/1e9:7.2f} G samples/s  {r['ms_per_step']:9.3f} ms/step  frac {r['roofline']['frac']:.3f}  clk {r['clocks'].get('sm_mhz')}")
except Exception as e:
    print(c, "FAILED", e, open(f"gpurun_out/qb_{c}.err").read()[-1500:])
PY
done
