#!/bin/bash
# round-2 evidence refresh after the eval / binning changes (render kernel
# unchanged): GPU suite, smoke, the default bench line, its ncu launch list,
# one device-timed line per config
python -m pytest tests -m gpu -q > gpurun_out/r2r_gputest.log 2>&1; tail -1 gpurun_out/r2r_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r2r_bench.json 2> gpurun_out/r2r_bench.err; python -c "
import json; r=json.load(open('gpurun_out/r2r_bench.json')); print('bench', r['value']/1e9, r['roofline']['frac'], r['e2e']['value']/1e9, r['eval']['value']/1e9, r['clocks'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2r_bench_c5_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r2r_ncu_launch.log 2>&1; tail -1 gpurun_out/r2r_ncu_launch.log
timeout 1200 python bench.py --all-configs --steps 3 --warmup 3 > gpurun_out/r2r_all_configs.jsonl 2> gpurun_out/r2r_all_configs.err
python - <<'PY'
import json
for l in open("gpurun_out/r2r_all_configs.jsonl"):
    x = json.loads(l)
    print(x["config"]["workload"], round(x["value"] / 1e9, 2), "G/s frac", round(x["roofline"]["frac"], 3), "fps", round(x.get("frames_per_s", 0), 1))
PY
