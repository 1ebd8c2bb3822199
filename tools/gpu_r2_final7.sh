#!/bin/bash
# round-2 HEAD evidence (final kernel + 8x4 quad warp units on grouped Bezier blocks):
# C5 bench launch, one line per config
python -m paper_2204_11762_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err; python -c "
import json; r=json.load(open('gpurun_out/r2i_bench.json')); print('bench', r['value']/1e9, r['roofline']['frac'], r['roofline']['north_star']['frac'], r['e2e']['value']/1e9, r['eval']['value']/1e9, r['clocks'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2i_bench_c5_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r2i_ncu_launch.log 2>&1; tail -1 gpurun_out/r2i_ncu_launch.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:render_kernel -c 1 -o gpurun_out/r2i_prof_c5 \
    python bench.py --workload c5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-eval > gpurun_out/r2i_ncu_c5.log 2>&1; tail -1 gpurun_out/r2i_ncu_c5.log
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/r2i_gputest.log 2>&1; grep -E "passed|failed" gpurun_out/r2i_gputest.log | tail -1
grep -E "^FAILED" gpurun_out/r2i_gputest.log | head -20
timeout 1200 python bench.py --all-configs --steps 3 --warmup 3 > gpurun_out/r2i_all_configs.jsonl 2> gpurun_out/r2i_all_configs.err
python - <<'PY'
import json
for l in open("gpurun_out/r2i_all_configs.jsonl"):
    x = json.loads(l)
    print(x["config"]["workload"], round(x["value"] / 1e9, 2), "G/s frac", round(x["roofline"]["frac"], 3), "fps", round(x.get("frames_per_s", 0), 1))
PY
timeout 900 python bench.py --emulate 8 > gpurun_out/r2i_emulate_c5.json 2> gpurun_out/r2i_emulate_c5.err; tail -c 300 gpurun_out/r2i_emulate_c5.json
