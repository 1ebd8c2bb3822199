#!/bin/bash
# round 2 diagnostic: C5 render with no block reloads / with every reload an L1 hit (wrong images)
for f in "" "-DMFA_DIAG_NORELOAD=1" "-DMFA_DIAG_L1=1" ""; do
  echo "=== flags: $f"
  MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  ./tools/quickbench.sh c5
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
