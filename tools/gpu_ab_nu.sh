#!/bin/bash
# round 2 A/B: span crossings on the shifted 32-bit offset (MFA_NU_SHIFTCMP) and
# a prefetch of the predicted next Bezier block (MFA_PREFETCH_NEXT 1 = L1, 2 = L2)
for f in "" "-DMFA_NU_SHIFTCMP=1" "-DMFA_NU_SHIFTCMP=1 -DMFA_PREFETCH_NEXT=1" "-DMFA_NU_SHIFTCMP=1 -DMFA_PREFETCH_NEXT=2" "-DMFA_PREFETCH_NEXT=1" ""; do
  echo "=== flags: $f"
  MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  ./tools/quickbench.sh c5
  if [ "$f" = "-DMFA_NU_SHIFTCMP=1" ]; then
    python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "subset or nonuniform or narrower or degrees or layouts or skip" 2>&1 | tail -2
  fi
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
