python -m paper_2204_11762_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "render or layouts or knots" 2>&1 | tail -2
./tools/quickbench.sh c5
echo "=== nu3 off"; MFA_EXTRA_NVCC_FLAGS="-DMFA_NU3=0" python -m paper_2204_11762_b200.build > /dev/null 2>&1; ./tools/quickbench.sh c5
python -m paper_2204_11762_b200.build > /dev/null 2>&1
