#!/bin/bash
# round 2: A/B (alternating) of the grouped Bezier layout (MFA_BEZ_GROUP=4); image hashes must match
for f in "" "-DMFA_BEZ_GROUP=4" "" "-DMFA_BEZ_GROUP=4"; do
  echo "=== flags: $f"
  MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  python tools/img_hash.py 2 5
  ./tools/quickbench.sh c5 c2
  python tools/eval_bench.py 5 2>&1 | tail -1
done
MFA_EXTRA_NVCC_FLAGS="-DMFA_BEZ_GROUP=4" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -m paper_2204_11762_b200.build > /dev/null 2>&1
