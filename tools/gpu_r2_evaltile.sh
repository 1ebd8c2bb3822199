#!/bin/bash
# round 2: binned eval with the bin's control-point tile staged in shared memory
python -m pytest tests -m gpu -x -q -k "eval or hessian or layouts or degrees" > gpurun_out/r2_evaltile_tests.log 2>&1; tail -2 gpurun_out/r2_evaltile_tests.log
for f in "" "-DMFA_EVAL_TILE=0" "-DMFA_EVAL_TILE=0 -DMFA_EVAL_CELLS=0" ""; do
  echo "=== flags: $f"
  MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  python tools/eval_bench.py 3 4 5 2>&1 | tail -3
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
M=gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active,launch__registers_per_thread,smsp__inst_executed.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active
ncu --metrics $M --clock-control none -k regex:"eval_" -c 1 --csv python tools/eval_bench.py 3 2>/dev/null | grep -E "eval_" | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' | cut -c1-150
