# Full GPU verification: build, smoke, all -m gpu tests, quick C3/C4/C5 bench
python -m paper_2204_11762_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rf ${PYTEST_K:+-k "$PYTEST_K"} -s > gpurun_out/gpu_tests.log 2>&1; grep -E "passed|failed" gpurun_out/gpu_tests.log | tail -3
grep -E "^FAILED|Error" gpurun_out/gpu_tests.log | head -20
./tools/quickbench.sh ${QB_WL:-c5}
