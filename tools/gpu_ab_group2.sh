#!/bin/bash
# round 2: eval on the grouped Bezier layout with w-fastest cells, vs linear
for f in "" "-DMFA_BEZ_GROUP=4"; do
  echo "=== flags: $f"
  MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  python tools/eval_bench.py 5 2 2>&1 | tail -2
  python tools/hess_bench.py 5 2>&1 | tail -1
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
