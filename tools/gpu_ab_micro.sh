# A/B of the render micro-optimisations (cubic Bernstein written out, ftz pow, int cache key)
python -m paper_2204_11762_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "render or layouts" 2>&1 | tail -2
./tools/quickbench.sh c5 c3 c4
for f in "-DMFA_BERN3=0" "-DMFA_FAST_POW=0" "-DMFA_BERN3=0 -DMFA_FAST_POW=0"; do
  echo "=== $f"; MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/build_variant.log 2>&1 || { tail gpurun_out/build_variant.log; continue; }
  ./tools/quickbench.sh c5
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
