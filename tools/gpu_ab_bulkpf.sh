#!/bin/bash
# A/B: bulk async prefetch of the sample-after-next's Bezier block into shared memory
for f in "-DMFA_BULK_PF=1" "" "-DMFA_BULK_PF=1"; do
  echo "=== flags: $f"
  MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  ./tools/quickbench.sh c5
  if [ "$f" = "-DMFA_BULK_PF=1" ]; then
    timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "subset or nonuniform or narrower or degrees or skip or both_layouts" 2>&1 | tail -2
  fi
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
