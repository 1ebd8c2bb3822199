#!/bin/bash
for f in "-DMFA_MACRO_LOG=1" "-DMFA_MACRO_LOG=2" "-DMFA_MACRO_LOG=3" "-DMFA_MACRO_LOG=0"; do
  echo "=== flags: $f"
  MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  QB_ARGS="--skip-transparent-blocks" ./tools/quickbench.sh c5
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
