#!/bin/bash
# round 2: the grouped Bezier layout as the AUTO default: full -m gpu suite, image hashes, quick bench, eval
python -m paper_2204_11762_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
python tools/img_hash.py 2 5
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/gpu_tests.log 2>&1; grep -E "passed|failed" gpurun_out/gpu_tests.log | tail -2
grep -E "^FAILED" gpurun_out/gpu_tests.log | head -20
./tools/quickbench.sh c5 c2 c3
python tools/eval_bench.py 5 2 3 2>&1 | tail -3
