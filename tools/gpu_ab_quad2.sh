#!/bin/bash
# the 2x2-lane-quad default: GPU suite; then A/B (alternating) of the 8x4 unit with 2x2 quads (MFA_UNIT_SHAPE=5) on C5
python -m paper_2204_11762_b200.build > gpurun_out/q2_build.log 2>&1 || { tail -20 gpurun_out/q2_build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/q2_gputest.log 2>&1; grep -E "passed|failed" gpurun_out/q2_gputest.log | tail -1
for f in "-DMFA_UNIT_SHAPE=5" "" "-DMFA_UNIT_SHAPE=5" ""; do
  echo "=== flags: $f"
  MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  python tools/img_hash.py 5
  ./tools/quickbench.sh c5
done
