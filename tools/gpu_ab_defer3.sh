#!/bin/bash
# round 2: A/B (alternating) of the shading before the multi-span vote (MULTI_DEFER=3); image hashes must match
for f in "-DMFA_MULTI_DEFER=3" "" "-DMFA_MULTI_DEFER=3" ""; do
  echo "=== flags: $f"
  MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  python tools/img_hash.py 5
  ./tools/quickbench.sh c5
done
timeout 900 python -m pytest tests -m gpu -x -q -k "subset or nonuniform or narrower or degrees or skip or both_layouts or mfa_render or multiple_knots or ert or tiled or scatter" 2>&1 | tail -2
