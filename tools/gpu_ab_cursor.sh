for b in 1 8 32; do echo "=== cursor stride $b"; MFA_EXTRA_NVCC_FLAGS="-DMFA_CURSOR_STRIDE=$b" python -m paper_2204_11762_b200.build > /dev/null 2>&1; python tools/eval_layouts.py 2>&1 | grep grad=True; done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
