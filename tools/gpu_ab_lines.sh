#!/bin/bash
# A/B: line-group slots for the binned p = 3 quad eval (MFA_EVAL_LINES), C3 2^24 points; eval GPU tests
M=gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,dram__bytes_read.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
python -m paper_2204_11762_b200.build > gpurun_out/ln_build1.log 2>&1 || { tail -20 gpurun_out/ln_build1.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "eval" > gpurun_out/ln_tests.log 2>&1; tail -3 gpurun_out/ln_tests.log
echo "== LINES=1"; python tools/eval_bench.py 3 5; python tools/eval_bench.py 3
timeout 600 ncu --metrics $M --clock-control none -k regex:eval -c 1 python tools/eval_bench.py 3 2>&1 | grep -E "eval_|gpu__time|wavefronts|dram__bytes|inst_executed|issue" | head -10
MFA_EXTRA_NVCC_FLAGS="-DMFA_EVAL_LINES=0" python -m paper_2204_11762_b200.build > gpurun_out/ln_build0.log 2>&1 || { tail -20 gpurun_out/ln_build0.log; exit 1; }
echo "== LINES=0"; python tools/eval_bench.py 3 5; python tools/eval_bench.py 3
