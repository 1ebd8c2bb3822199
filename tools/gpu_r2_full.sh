#!/bin/bash
# full round-2 validation: every -m gpu test, smoke, the default bench line
python -m pytest tests -m gpu -q > gpurun_out/r2_gputest_full.log 2>&1; tail -3 gpurun_out/r2_gputest_full.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/r2_bench_default.json 2> gpurun_out/r2_bench_default.err; python -c "
import json; r=json.load(open('gpurun_out/r2_bench_default.json'))
print('value', r['value']/1e9, 'frac', r['roofline']['frac'], 'e2e', r['e2e']['value']/1e9, 'cpu', r['cpu_baseline']['value']/1e6, 'clocks', r['clocks'])"
