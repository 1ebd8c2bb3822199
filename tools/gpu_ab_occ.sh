#!/bin/bash
# round 2: occupancy variants of the C5 render with the final kernel (alternating with the default)
for f in "" "-DMFA_RENDER_THREADS=64 -DMFA_RENDER_MAXNREG=144 -DMFA_RENDER_MINB=7" "-DMFA_RENDER_THREADS=32 -DMFA_RENDER_MAXNREG=152 -DMFA_RENDER_MINB=13" "-DMFA_RENDER_THREADS=128 -DMFA_RENDER_MAXNREG=128 -DMFA_RENDER_MINB=4" "" "-DMFA_RENDER_THREADS=64 -DMFA_RENDER_MAXNREG=144 -DMFA_RENDER_MINB=7"; do
  echo "=== flags: $f"
  MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  python tools/img_hash.py 5
  ./tools/quickbench.sh c5
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
