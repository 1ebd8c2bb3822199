#!/bin/bash
# compute-sanitizer is closed on this pool: the bounds-checked build instead
# (-DMFA_DEBUG_BOUNDS: MFA_DCHECK traps on an out-of-range block / span /
# record / TF / macro-block index) over tools/sanitize_small.py (every entry
# point, all layouts, shading modes 0-3, host-buffer renders, IPC buffer) and
# the GPU suite
MFA_EXTRA_NVCC_FLAGS="-DMFA_DEBUG_BOUNDS" python -m paper_2204_11762_b200.build > gpurun_out/san_build.log 2>&1 || { tail -5 gpurun_out/san_build.log; exit 1; }
timeout 1200 python tools/sanitize_small.py > gpurun_out/san_small.log 2>&1; echo "sanitize_small rc=$?"; tail -3 gpurun_out/san_small.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/san_gputest.log 2>&1; echo "gpu suite rc=$?"; tail -2 gpurun_out/san_gputest.log
grep -c "MFA_DCHECK failed" gpurun_out/san_small.log gpurun_out/san_gputest.log
python -m paper_2204_11762_b200.build > /dev/null 2>&1
