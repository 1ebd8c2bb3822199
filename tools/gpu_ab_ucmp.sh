#!/bin/bash
for f in "-DMFA_NU_UCMP=1" "" "-DMFA_NU_UCMP=1" ""; do
  echo "=== flags: $f"
  MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  ./tools/quickbench.sh c5
done
MFA_EXTRA_NVCC_FLAGS="-DMFA_NU_UCMP=1" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "subset or nonuniform or narrower or degrees or skip or both_layouts or hessian or quality" 2>&1 | tail -2
python -m paper_2204_11762_b200.build > /dev/null 2>&1
