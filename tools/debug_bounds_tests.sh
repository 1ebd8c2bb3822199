#!/bin/bash
# Rebuild with device bounds checks and run the GPU suite + the small sanitizer workload, then restore.
MFA_EXTRA_NVCC_FLAGS="-DMFA_DEBUG_BOUNDS" python -m paper_2204_11762_b200.build > gpurun_out/build_debug.log 2>&1 || { tail gpurun_out/build_debug.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_debug.log 2>&1; rc=$?
echo "debug-bounds pytest rc=$rc"; tail -3 gpurun_out/pytest_gpu_debug.log
python tools/sanitize_small.py > gpurun_out/debug_small.log 2>&1; echo "debug-bounds small rc=$?"; grep -c DCHECK gpurun_out/*.log
python -m paper_2204_11762_b200.build > /dev/null 2>&1
