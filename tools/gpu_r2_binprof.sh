#!/bin/bash
# round 2: ncu --set full of the binning kernels (count, scatter, gather) on C3 2^24 points
timeout 900 ncu --set full --clock-control none -k regex:"bin_count|bin_scatter|bin_gather" -c 3 -o gpurun_out/r2_binprof python tools/eval_bench.py 3 > gpurun_out/r2_binprof.log 2>&1; tail -2 gpurun_out/r2_binprof.log
