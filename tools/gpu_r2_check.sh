#!/bin/bash
# round-end check of the committed state: GPU suite, smoke, default bench line,
# the reference (oracle) arm
python -m pytest tests -m gpu -q > gpurun_out/r2c_gputest.log 2>&1; tail -2 gpurun_out/r2c_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err; cut -c1-300 gpurun_out/r2c_bench.json; echo
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2c_ref.json 2> gpurun_out/r2c_ref.err; cut -c1-300 gpurun_out/r2c_ref.json
