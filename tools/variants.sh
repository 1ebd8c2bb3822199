#!/bin/bash
# Build-flag sweep: for each quoted flag set, rebuild libmfa.so and run the quick bench.
# usage: tools/variants.sh "FLAGS1" "FLAGS2" ...   (workloads from $WL, default "c3 c4 c5")
for f in "$@"; do
  echo "=== flags: $f"
  MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/build_variant.log 2>&1 || { echo build failed; tail gpurun_out/build_variant.log; continue; }
  ./tools/quickbench.sh ${WL:-c3 c4 c5}
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
