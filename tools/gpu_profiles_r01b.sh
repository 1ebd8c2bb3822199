# round-1 profile refresh: bench launch list (same command as the driver's bench), full captures of
# the render kernel (C5, 2 views), eval (C3), hessian (C3), SSIM, field render
set -x
python -m paper_2204_11762_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch_b.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:eval_kernel -c 1 -o gpurun_out/prof_eval_c3 python tools/profile_render.py c3 --eval --reps 1 > gpurun_out/ncu_eval.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hessian_kernel -c 1 -o gpurun_out/prof_hess_c3 python tools/profile_hessian.py > gpurun_out/ncu_hess.log 2>&1
tail -2 gpurun_out/ncu_eval.log gpurun_out/ncu_hess.log
