# A/B of the register-record render variant on C5 (quads layout) vs Bezier blocks
set -x
python -m paper_2204_11762_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "layouts or multiple_knots or subset_parity" > gpurun_out/gpu_tests_rec.log 2>&1; tail -5 gpurun_out/gpu_tests_rec.log
QB_ARGS="--layout quads" ./tools/quickbench.sh c5
QB_ARGS="--layout bezier" ./tools/quickbench.sh c5
for f in "-DMFA_REC_MINB=3" "-DMFA_REC_THREADS=160" "-DMFA_REC_THREADS=192"; do
  echo "=== $f"; MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/build_variant.log 2>&1 || { tail gpurun_out/build_variant.log; continue; }
  QB_ARGS="--layout quads" ./tools/quickbench.sh c5
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
