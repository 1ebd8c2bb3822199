#!/bin/bash
# round 2: A/B (alternating) of the binning / gather ILP (points per thread per iteration)
python -m pytest tests -m gpu -x -q -k "eval or hessian" 2>&1 | tail -2
for f in "" "-DMFA_BIN_ILP=1" "-DMFA_BIN_ILP=8" "" "-DMFA_BIN_ILP=1" "-DMFA_BIN_ILP=8"; do
  echo "=== flags: $f"
  MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  python tools/eval_bench.py 3 5 2>&1 | tail -2
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bin_|eval_" -c 6 --csv python tools/eval_bench.py 3 2>/dev/null | grep -E "gpu__time" | awk -F'","' '{print $5, $(NF-1), $NF}' | cut -c1-120
