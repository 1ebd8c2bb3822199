for f in "-DMFA_CARVEOUT=8" "-DMFA_CARVEOUT=16" "-DMFA_CARVEOUT=25"; do
  echo "=== $f"; MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > /dev/null 2>&1; ./tools/quickbench.sh c5 c3 c4
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
