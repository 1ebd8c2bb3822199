python -m paper_2204_11762_b200.build > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
./tools/quickbench.sh c4 c3 c5
