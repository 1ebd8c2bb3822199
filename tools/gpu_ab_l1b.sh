python -m paper_2204_11762_b200.build > gpurun_out/build.log 2>&1 || exit 1
./tools/quickbench.sh c5 c3 c4
echo "=== fixed 25"; MFA_EXTRA_NVCC_FLAGS="-DMFA_CARVEOUT=25" python -m paper_2204_11762_b200.build > /dev/null 2>&1; ./tools/quickbench.sh c4
echo "=== driver default (100 = max smem)"; MFA_EXTRA_NVCC_FLAGS="-DMFA_CARVEOUT=100" python -m paper_2204_11762_b200.build > /dev/null 2>&1; ./tools/quickbench.sh c5 c3 c4
python -m paper_2204_11762_b200.build > /dev/null 2>&1
