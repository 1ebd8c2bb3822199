for f in "-DMFA_BEZ_HALF=1 -DMFA_RENDER_MINB=4" "-DMFA_BEZ_HALF=1"; do
  echo "=== $f"; MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > /dev/null 2>&1; ./tools/quickbench.sh c5
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
