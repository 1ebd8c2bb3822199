#!/bin/bash
python -m pytest tests -m gpu -q > gpurun_out/r2g_gputest.log 2>&1; tail -2 gpurun_out/r2g_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py --all-configs --steps 3 --warmup 3 > gpurun_out/r2g_all_configs.jsonl 2> gpurun_out/r2g_all_configs.err
python - <<'PY'
import json
for l in open("gpurun_out/r2g_all_configs.jsonl"):
    x = json.loads(l)
    print(x["config"]["workload"], round(x["value"] / 1e9, 2), "G/s frac", round(x["roofline"]["frac"], 3), "fps", round(x["frames_per_s"], 1))
PY
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; python -c "
import json; r=json.load(open('gpurun_out/r2g_bench.json')); print('bench', r['value']/1e9, r['roofline']['frac'], r['e2e']['value']/1e9, r['eval']['value']/1e9)"
