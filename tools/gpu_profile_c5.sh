set -x
python -m paper_2204_11762_b200.build > gpurun_out/build.log 2>&1
QB_ARGS="--layout quads" ./tools/quickbench.sh c5 > gpurun_out/qb_quads.txt 2>&1
cat gpurun_out/qb_quads.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_kernel -c 1 -o gpurun_out/prof_c5_v5 python tools/profile_render.py c5 --views 2 --reps 1 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_launch.log 2>&1
tail -2 gpurun_out/ncu_launch.log
