for f in "-DMFA_BEZ_CACHE=0" "-DMFA_BEZ_CACHE=0 -DMFA_RENDER_MINB=4" "-DMFA_BEZ_CACHE=0 -DMFA_RENDER_THREADS=256 -DMFA_RENDER_MINB=2"; do
  echo "=== $f"; MFA_EXTRA_NVCC_FLAGS="$f" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; continue; }
  cuobjdump -res-usage paper_2204_11762_b200/build/render.cu.o 2>&1 | grep -A1 "ILi3ELi1ELb0ELb1ELb0" | grep REG
  ./tools/quickbench.sh c5
done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
