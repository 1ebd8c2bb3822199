# A/B: make the next sample's contraction wait on the shading of the current one
# (MFA_ORDER 1: on A after compositing, 2: on the TF opacity, 3: on the TF colour)
python -m paper_2204_11762_b200.build > gpurun_out/build.log 2>&1 || exit 1
./tools/quickbench.sh c5 c3
for o in 1 2 3; do
  echo "=== MFA_ORDER=$o"; MFA_EXTRA_NVCC_FLAGS="-DMFA_ORDER=$o" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  ./tools/quickbench.sh c5 c3
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
