# A/B: pixel shape of a warp's 32-ray unit (MFA_UNIT_SHAPE: 0 = 8x4, 1 = 4x8, 2 = 16x2), alternated twice
for rep in 1 2; do
  python -m paper_2204_11762_b200.build > gpurun_out/build.log 2>&1 || exit 1
  echo "=== 8x4"; ./tools/quickbench.sh c5 c3
  MFA_EXTRA_NVCC_FLAGS="-DMFA_UNIT_SHAPE=1" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || exit 1
  echo "=== 4x8"; ./tools/quickbench.sh c5 c3
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
