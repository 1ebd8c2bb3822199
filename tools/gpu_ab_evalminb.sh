for mb in 1 4 5 6; do echo "=== minb $mb"; MFA_EXTRA_NVCC_FLAGS="-DMFA_EVAL_MINB=$mb" python -m paper_2204_11762_b200.build > /dev/null 2>&1; python tools/eval_layouts.py; done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
