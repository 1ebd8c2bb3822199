#!/bin/bash
# round-2 re-entry check at HEAD: build, smoke, every -m gpu test, the default bench line
python -m paper_2204_11762_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/r2h_gputest.log 2>&1; grep -E "passed|failed" gpurun_out/r2h_gputest.log | tail -1
grep -E "^FAILED" gpurun_out/r2h_gputest.log | head -20
timeout 900 python bench.py > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err; python -c "
import json; r=json.load(open('gpurun_out/r2h_bench.json')); print('bench', r['value']/1e9, r['roofline']['frac'], r['e2e']['value']/1e9, r['eval']['value']/1e9, r['clocks'])"
