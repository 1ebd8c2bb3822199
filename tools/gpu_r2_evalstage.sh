#!/bin/bash
# round 2: eval with the bin's control points staged in shared memory (uniform quads)
python -m pytest tests -m gpu -x -q -k "eval or hessian or layouts or degrees" > gpurun_out/r2_evalstage_tests.log 2>&1; tail -2 gpurun_out/r2_evalstage_tests.log
for f in "" "-DMFA_EVAL_STAGE_THREADS=256" "-DMFA_EVAL_STAGE_THREADS=64" "-DMFA_EVAL_STAGE=0"; do
  echo "=== flags: $f"
  MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  python tools/eval_bench.py 3 2 2>&1 | tail -2
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum --clock-control none -k regex:"eval_|bin_" -c 6 --csv python tools/eval_bench.py 3 2>/dev/null | grep -E "gpu__time|dram__bytes|wavefronts|inst_exec" | awk -F'","' '{print $5, $(NF-2), $(NF-1), $NF}' | cut -c1-150
