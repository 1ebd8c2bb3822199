#!/bin/bash
# round-2 (session 3) evidence: the default bench line and its ncu launch list
python -m paper_2204_11762_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err; python -c "
import json; r=json.load(open('gpurun_out/r2s_bench.json')); print('bench', r['value']/1e9, r['roofline']['frac'], r['e2e']['value']/1e9, r['eval']['value']/1e9, r['clocks'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2s_bench_c5_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r2s_ncu_launch.log 2>&1; tail -1 gpurun_out/r2s_ncu_launch.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2s_ref.json 2> gpurun_out/r2s_ref.err; tail -c 300 gpurun_out/r2s_ref.json
