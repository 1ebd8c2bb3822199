#!/bin/bash
# final round-2 evidence with the final build: GPU suite, smoke, bench default,
# all-config lines, emulation, bench --gpus 2 (shared GPU), ncu launch list +
# one --set full capture of the bench's render launch
python -m pytest tests -m gpu -q > gpurun_out/r2f_gputest.log 2>&1; tail -2 gpurun_out/r2f_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; tail -c 400 gpurun_out/r2f_bench.json; echo
timeout 1200 python bench.py --all-configs --steps 3 --warmup 3 > gpurun_out/r2f_all_configs.jsonl 2> gpurun_out/r2f_all_configs.err; cut -c1-160 gpurun_out/r2f_all_configs.jsonl
timeout 900 python bench.py --emulate 8 --steps 1 > gpurun_out/r2f_emulate_c5.json 2> gpurun_out/r2f_emulate_c5.err; cut -c1-400 gpurun_out/r2f_emulate_c5.json
timeout 900 python bench.py --gpus 2 --steps 2 --warmup 3 --no-eval --no-cpu-baseline > gpurun_out/r2f_bench_g2.json 2> gpurun_out/r2f_bench_g2.err; cut -c1-300 gpurun_out/r2f_bench_g2.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2f_bench_c5_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r2f_ncu_launch.log 2>&1; tail -1 gpurun_out/r2f_ncu_launch.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:render_kernel -c 1 -o gpurun_out/r2f_prof_c5 \
    python bench.py --workload c5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-eval > gpurun_out/r2f_ncu_c5.log 2>&1; tail -1 gpurun_out/r2f_ncu_c5.log
