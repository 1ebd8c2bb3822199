python -m paper_2204_11762_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_quality.py -q -k "render or layouts or knots or lights or field or degrees or multiview or tiled" 2>&1 | tail -3
./tools/quickbench.sh c5
for f in "-DMFA_NU32_INLINE=1" "-DMFA_NU_T32=0"; do
  echo "=== $f"; MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > /dev/null 2>&1; ./tools/quickbench.sh c5
done
echo "=== inline parity"; MFA_EXTRA_NVCC_FLAGS="-DMFA_NU32_INLINE=1" python -m paper_2204_11762_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "subset_parity or layouts or knots" 2>&1 | tail -2
python -m paper_2204_11762_b200.build > /dev/null 2>&1
