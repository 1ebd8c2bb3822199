#!/bin/bash
# round 2 diagnostic: the C5 render without the multi-span crossing loop (wrong images where a step
# crosses several spans) -- what the multi-span handling costs
for f in "" "-DMFA_DIAG_NOMULTI=1" ""; do
  echo "=== flags: $f"
  MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  ./tools/quickbench.sh c5
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
