#!/bin/bash
# round 2: eval (AoS results at the original index + transpose) and render occupancy A/B
python -m pytest tests -m gpu -x -q -k "eval or hessian" > gpurun_out/r2_evaltests.log 2>&1; tail -2 gpurun_out/r2_evaltests.log
python tools/eval_bench.py 3 5 2>&1 | tail -3
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"eval_kernel|bin_|aos_" -c 6 --csv python tools/eval_bench.py 3 2>/dev/null | grep -E "gpu__time|dram__bytes" | awk -F'","' '{print $5, $(NF-2), $(NF-1), $NF}' | cut -c1-160
for f in "" "-DMFA_RENDER_THREADS=32 -DMFA_RENDER_MAXNREG=152 -DMFA_RENDER_MINB=13" "-DMFA_RENDER_THREADS=32 -DMFA_RENDER_MAXNREG=144 -DMFA_RENDER_MINB=14" "-DMFA_RENDER_THREADS=32 -DMFA_RENDER_MINB=12"; do
  echo "=== flags: $f"
  MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  ./tools/quickbench.sh c5 c3
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
