#!/bin/bash
# A/B (alternating) on C5: 16x2 unit with 2x2-lane quads (MFA_UNIT_SHAPE=6) vs the default (grouped Bezier: 8x4 with quads)
for f in "-DMFA_UNIT_SHAPE=6" "" "-DMFA_UNIT_SHAPE=6" ""; do
  echo "=== flags: $f"
  MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  python tools/img_hash.py 5
  ./tools/quickbench.sh c5
done
