#!/bin/bash
# round 2: grouped Bezier layout -- group shapes (log2 extents u,v,w: 0=(0,0,2) 1=(0,1,1) 2=(1,0,1) 3=(2,0,0) 4=(1,1,0))
for f in "-DMFA_BEZ_GSHAPE=0" "" "-DMFA_BEZ_GSHAPE=3" "-DMFA_BEZ_GSHAPE=4" "" "-DMFA_BEZ_GSHAPE=0"; do
  echo "=== flags: $f"
  MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  python tools/img_hash.py 5
  ./tools/quickbench.sh c5
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
