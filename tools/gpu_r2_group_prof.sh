#!/bin/bash
# round 2: grouped Bezier layout -- full -m gpu suite, ncu --set full of the C5 render (4 views), unit / view-group A/B
python -m paper_2204_11762_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/gpu_tests.log 2>&1; grep -E "passed|failed" gpurun_out/gpu_tests.log | tail -1
grep -E "^FAILED" gpurun_out/gpu_tests.log | head -20
timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_kernel -c 1 -o gpurun_out/r2g_prof_c5v4 \
    python tools/profile_render.py c5 --views 4 --reps 1 > gpurun_out/r2g_ncu.log 2>&1; tail -2 gpurun_out/r2g_ncu.log
for f in "-DMFA_UNIT_SHAPE=0" "" "-DMFA_VIEW_GROUP=2" "-DMFA_VIEW_GROUP=8" ""; do
  echo "=== flags: $f"
  MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  ./tools/quickbench.sh c5
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
