#!/bin/bash
# cells-on-quads diagnostics: full ncu capture of eval_cells_kernel (C3), and CTA-size variants
MFA_EXTRA_NVCC_FLAGS="-DMFA_EVAL_CELLS_QUADS=1" python -m paper_2204_11762_b200.build > gpurun_out/cq2_build.log 2>&1 || { tail -20 gpurun_out/cq2_build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:eval_cells -c 1 -o gpurun_out/cq2_cells python tools/eval_bench.py 3 > gpurun_out/cq2_ncu.log 2>&1; tail -2 gpurun_out/cq2_ncu.log
for T in 256 512; do
  MFA_EXTRA_NVCC_FLAGS="-DMFA_EVAL_CELLS_QUADS=1 -DMFA_CELL_THREADS=$T" python -m paper_2204_11762_b200.build > gpurun_out/cq2_build$T.log 2>&1 || { tail -20 gpurun_out/cq2_build$T.log; exit 1; }
  echo "== threads $T"; python tools/eval_bench.py 3; python tools/eval_bench.py 3
done
