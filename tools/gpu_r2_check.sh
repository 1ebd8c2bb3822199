#!/bin/bash
# round-2 GPU check: the -m gpu suite, the 1-GPU rank emulation (C5, 8 ranks),
# bench --gpus 2 on one GPU (functional), the default bench line
python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest.log 2>&1; tail -3 gpurun_out/r2_gputest.log
timeout 900 python bench.py --emulate 8 --steps 1 > gpurun_out/r2_emulate_c5.json 2> gpurun_out/r2_emulate_c5.err; tail -c 3000 gpurun_out/r2_emulate_c5.json; tail -3 gpurun_out/r2_emulate_c5.err
timeout 900 python bench.py --emulate 8 --steps 2 --workload c4 > gpurun_out/r2_emulate_c4.json 2> gpurun_out/r2_emulate_c4.err; tail -c 2000 gpurun_out/r2_emulate_c4.json
timeout 900 python bench.py --gpus 2 --steps 2 --warmup 3 --no-eval --no-cpu-baseline > gpurun_out/r2_bench_g2.json 2> gpurun_out/r2_bench_g2.err; tail -c 1500 gpurun_out/r2_bench_g2.json; tail -5 gpurun_out/r2_bench_g2.err
timeout 900 python bench.py --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; tail -c 1200 gpurun_out/r2_bench.json; tail -3 gpurun_out/r2_bench.err
