#!/bin/bash
# A/B of two prebuilt libraries (gpurun_out/ab/libmfa_{base,new}.so), alternating
for v in base new base new; do
  cp gpurun_out/ab/libmfa_$v.so paper_2204_11762_b200/libmfa.so; touch paper_2204_11762_b200/libmfa.so
  echo "=== $v"; ./tools/quickbench.sh ${WL:-c5}
done
cp gpurun_out/ab/libmfa_new.so paper_2204_11762_b200/libmfa.so; touch paper_2204_11762_b200/libmfa.so
