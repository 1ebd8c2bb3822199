#!/bin/bash
# A/B (alternating): warp unit 4x8 with 2x2-pixel 4-lane groups (MFA_UNIT_SHAPE=4) vs 4x1 rows (1);
# the L1 data pipe serves an LDG.256 in groups of 4 lanes. Image hashes must match.
for f in "-DMFA_UNIT_SHAPE=4" "" "-DMFA_UNIT_SHAPE=4" ""; do
  echo "=== flags: $f"
  MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  python tools/img_hash.py 5
  ./tools/quickbench.sh c5 c3 c4
done
