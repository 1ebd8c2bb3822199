python -m paper_2204_11762_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_quality.py -q -k "render or layouts or knots or lights or field" 2>&1 | tail -2
./tools/quickbench.sh c5
QB_ARGS="--layout quads" ./tools/quickbench.sh c5
echo "=== no span records"; MFA_EXTRA_NVCC_FLAGS="-DMFA_SPAN_REC=0" python -m paper_2204_11762_b200.build > /dev/null 2>&1; ./tools/quickbench.sh c5
python -m paper_2204_11762_b200.build > /dev/null 2>&1
