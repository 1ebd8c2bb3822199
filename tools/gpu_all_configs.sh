# device-timed render throughput on every config (shaded and value-only), the final round-1 build
python -m paper_2204_11762_b200.build > gpurun_out/build.log 2>&1 || exit 1
echo "# shaded (bench.py --workload cN, 3 steps after 2 warm-up, device-timed)"
./tools/quickbench.sh c1 c2 c3 c4 c5
echo "# value-only (--no-shading)"
QB_ARGS="--no-shading" ./tools/quickbench.sh c3 c4 c5
echo "# eval (2^24 random points, binned)"
python tools/eval_bench.py 3 5
echo "# image quality"
python tools/quality_time.py
echo "# fit"
python tools/fit_time.py big
