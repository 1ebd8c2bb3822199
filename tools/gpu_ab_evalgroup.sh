#!/bin/bash
# round 2: eval on the grouped Bezier layout with group-ordered cells (C5 model), parity subset
python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; exit 1; }
for r in 1 2; do python tools/eval_bench.py 5 2 2>&1 | tail -2; python tools/hess_bench.py 5 2>&1 | tail -1; done
timeout 900 python -m pytest tests -m gpu -x -q -k "eval or hessian or both_layouts" 2>&1 | tail -2
