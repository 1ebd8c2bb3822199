python -m pytest tests -m gpu -x -q -k "eval or hessian or layouts or degrees" 2>&1 | tail -2
for f in "" "-DMFA_EVAL_CELLS=0" "" "-DMFA_EVAL_CELLS=0"; do
  echo "=== flags: $f"
  MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  python tools/eval_bench.py 3 4 5 2>&1 | tail -3
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
