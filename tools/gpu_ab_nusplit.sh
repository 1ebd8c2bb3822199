# A/B: non-uniform span crossings in two phases (issue the three axes' record loads, then consume)
python -m paper_2204_11762_b200.build > gpurun_out/build.log 2>&1 || exit 1
./tools/quickbench.sh c5
for f in "-DMFA_NU_SPLIT=1" "-DMFA_NU_SPLIT=2"; do
  echo "=== $f"; MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  ./tools/quickbench.sh c5
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
