#!/bin/bash
# C3 (256^3 uniform, p = 3) on the grouped / linear Bezier blocks (4.1 GB) vs the AUTO quads, with the HEAD kernel
python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; exit 1; }
for l in auto bezier_grouped bezier auto bezier_grouped; do
  echo "=== layout $l"; QB_ARGS="--layout $l" ./tools/quickbench.sh c3
done
