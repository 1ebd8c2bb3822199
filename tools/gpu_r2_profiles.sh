#!/bin/bash
# round-2 evidence: per-config bench lines, the launch list of the driver's
# bench command, --set full captures of the render on C5 (the bench launch),
# C4 and C3 (-> profiles/traffic.json), and of the binned eval on C3
timeout 1200 python bench.py --all-configs --steps 3 --warmup 3 > gpurun_out/r2_all_configs.jsonl 2> gpurun_out/r2_all_configs.err; cat gpurun_out/r2_all_configs.jsonl | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_bench_c5_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r2_ncu_launch.log 2>&1; tail -2 gpurun_out/r2_ncu_launch.log
for c in c5 c4 c3; do
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:render_kernel -c 1 -o gpurun_out/r2_prof_$c \
    python bench.py --workload $c --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-eval > gpurun_out/r2_ncu_$c.log 2>&1
  tail -2 gpurun_out/r2_ncu_$c.log
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"eval_kernel|bin_" -c 5 -o gpurun_out/r2_prof_eval_c3 python tools/eval_bench.py 3 > gpurun_out/r2_ncu_eval.log 2>&1; tail -2 gpurun_out/r2_ncu_eval.log
ls -la gpurun_out/*.ncu-rep
