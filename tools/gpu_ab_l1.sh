# A/B: shared-memory carveout (L1 size) and CTA-tile scheduling for p = 3
python -m paper_2204_11762_b200.build > gpurun_out/build.log 2>&1 || exit 1
./tools/quickbench.sh c5 c3
for f in "-DMFA_CARVEOUT=0" "-DMFA_CARVEOUT=10" "-DMFA_CARVEOUT=25" "-DMFA_CTA_TILES=1" "-DMFA_CTA_TILES=1 -DMFA_CARVEOUT=10"; do
  echo "=== $f"; MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/build_variant.log 2>&1 || { tail gpurun_out/build_variant.log; continue; }
  ./tools/quickbench.sh c5 c3
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
