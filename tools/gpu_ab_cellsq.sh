#!/bin/bash
# A/B: the bin cell sort on the quad layout (C3 eval, 2^24 points): time + L1 data-pipe wavefronts of the eval kernel
M=gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,dram__bytes_read.sum,smsp__inst_executed.sum,l1tex__t_sector_hit_rate.pct
for V in 0 1; do
  MFA_EXTRA_NVCC_FLAGS="-DMFA_EVAL_CELLS_QUADS=$V" python -m paper_2204_11762_b200.build > gpurun_out/cq_build$V.log 2>&1 || { tail -20 gpurun_out/cq_build$V.log; exit 1; }
  echo "== CELLS_QUADS=$V"
  python tools/eval_bench.py 3 4; python tools/eval_bench.py 3 4
  timeout 600 ncu --metrics $M --clock-control none -k regex:eval -c 2 python tools/eval_bench.py 3 2>&1 | grep -E "eval|gpu__time|wavefronts|dram__bytes|inst_executed|hit_rate" | head -20
done
