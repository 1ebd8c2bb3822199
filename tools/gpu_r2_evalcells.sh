#!/bin/bash
# round 2: binned eval with a per-bin cell sort in shared memory (eval_cells_kernel)
python -m pytest tests -m gpu -x -q -k "eval or hessian or layouts or degrees" > gpurun_out/r2_evalcells_tests.log 2>&1; tail -2 gpurun_out/r2_evalcells_tests.log
for f in "" "-DMFA_EVAL_CELLS=0" "" "-DMFA_EVAL_CELLS=0"; do
  echo "=== flags: $f"
  MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  python tools/eval_bench.py 3 5 2>&1 | tail -2
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts.sum,smsp__inst_executed.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"eval_|bin_" -c 6 --csv python tools/eval_bench.py 3 2>/dev/null | grep -E "gpu__time|dram__bytes|wavefronts|inst_exec|registers|warps_active" | awk -F'","' '{print $5, $(NF-2), $(NF-1), $NF}' | cut -c1-150
