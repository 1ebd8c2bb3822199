#!/bin/bash
# round 2: new-test subset, then device-timed lines for NEXT-1 (shaded / skip
# transparent gradient / value-only on C3, C4, C5) and the layouts of C5 / C3
python -m pytest tests -m gpu -x -q -k "bricks or skip_transparent or many_renders or entry_point or subset_parity or binned" > gpurun_out/r2_newtests.log 2>&1; tail -3 gpurun_out/r2_newtests.log
line() {  # workload, label, extra args
  timeout 900 python bench.py --workload $1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-eval $3 > gpurun_out/v_$1_$2.json 2> gpurun_out/v_$1_$2.err
  python - "$1" "$2" <<'PY'
import json,sys
c,l=sys.argv[1:3]
try:
    r=json.load(open(f"gpurun_out/v_{c}_{l}.json"))
    print(f"{c} {l:10s}: {r['value']/1e9:7.2f} G samples/s {r['ms_per_step']:9.3f} ms/step frac {r['roofline']['frac']:.3f} "
          f"layout {r['config']['layout']} footprint {r['config']['footprint_ratio']:.2f}x create {r['config']['create_ms']:.0f} ms clk {r['clocks'].get('sm_mhz')}")
except Exception as e:
    print(c, l, "FAILED", e, open(f"gpurun_out/v_{c}_{l}.err").read()[-1500:])
PY
}
for c in c3 c4 c5; do
  line $c shaded ""
  line $c skipgrad "--skip-transparent-gradient"
  line $c noshade "--no-shading"
done
line c5 bricks "--layout bricks"
line c5 quads "--layout quads"
line c3 bricks "--layout bricks"
line c2 bricks "--layout bricks"
line c2 shaded ""
