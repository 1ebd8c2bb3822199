#!/bin/bash
# round 2: A/B (alternating) of the Hessian gather ILP
python -m pytest tests -m gpu -x -q -k "hessian" 2>&1 | tail -1
for f in "" "-DMFA_HESS_ILP=1" "" "-DMFA_HESS_ILP=1"; do
  echo "=== flags: $f"
  MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  python tools/hess_bench.py 3 5 2>&1 | tail -2
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
