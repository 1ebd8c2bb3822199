#!/bin/bash
# round-2 (session 3) evidence: the grouped Bezier layout + 16-byte span records.
# GPU suite, smoke, --set full capture of the full C5 bench launch, per-config lines, 8-rank emulation
python -m paper_2204_11762_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/r2s_gputest.log 2>&1; grep -E "passed|failed" gpurun_out/r2s_gputest.log | tail -1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:render_kernel -c 1 -o gpurun_out/r2s_prof_c5 \
    python bench.py --workload c5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-eval > gpurun_out/r2s_ncu_c5.log 2>&1; tail -1 gpurun_out/r2s_ncu_c5.log
timeout 1200 python bench.py --all-configs --steps 3 --warmup 3 > gpurun_out/r2s_all_configs.jsonl 2> gpurun_out/r2s_all_configs.err
python - <<'PY'
import json
for l in open("gpurun_out/r2s_all_configs.jsonl"):
    x = json.loads(l)
    print(x["config"]["workload"], round(x["value"] / 1e9, 2), "G/s frac", round(x["roofline"]["frac"], 3), "fps", round(x.get("frames_per_s", 0), 1))
PY
timeout 900 python bench.py --emulate 8 > gpurun_out/r2s_emulate_c5.json 2> gpurun_out/r2s_emulate_c5.err; tail -c 400 gpurun_out/r2s_emulate_c5.json
