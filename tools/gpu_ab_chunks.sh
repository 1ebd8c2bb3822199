python -m paper_2204_11762_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "render or tiled or multiview or layouts" 2>&1 | tail -2
./tools/quickbench.sh c5 c3 c4
echo "=== chunks off"; MFA_EXTRA_NVCC_FLAGS="-DMFA_SM_CHUNKS=0" python -m paper_2204_11762_b200.build > /dev/null 2>&1; ./tools/quickbench.sh c5 c3 c4
python -m paper_2204_11762_b200.build > /dev/null 2>&1
