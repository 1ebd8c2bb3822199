for b in 8 6 4 2; do echo "=== bin spans $b"; MFA_EXTRA_NVCC_FLAGS="-DMFA_BIN_SPANS=$b" python -m paper_2204_11762_b200.build > /dev/null 2>&1; python tools/eval_layouts.py 2>&1 | grep grad=True; done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
