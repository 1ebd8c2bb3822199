python -m paper_2204_11762_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
./tools/quickbench.sh c3 c4 c5
QB_ARGS="--layout quads" ./tools/quickbench.sh c5
python tools/eval_layouts.py
