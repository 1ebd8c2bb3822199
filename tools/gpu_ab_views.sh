#!/bin/bash
# A/B (round 2): cross-view work order for the 64-view C5 batch:
# groups of orbit-adjacent views interleaved per supertile (ORDER 1) or per
# supertile row (ORDER 2), device-timed C5 + DRAM bytes / hit rates per launch.
M="dram__bytes_read.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,gpu__time_duration.sum"
run() {
  echo "=== flags: $1"
  MFA_EXTRA_NVCC_FLAGS="$1" python -m paper_2204_11762_b200.build > gpurun_out/bv.log 2>&1 || { tail -5 gpurun_out/bv.log; return; }
  ./tools/quickbench.sh c5
  timeout 300 ncu --metrics $M --clock-control none -k regex:render_kernel -c 1 --csv \
     python bench.py --workload c5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-eval 2>/dev/null \
     | grep -E '"(dram__bytes_read.sum|lts__t_sector_hit_rate.pct|l1tex__t_sector_hit_rate.pct|gpu__time_duration.sum)"' \
     | awk -F'","' '{print "   ", $(NF-2), $(NF-1), $NF}'
}
run ""
if [ $# -eq 0 ]; then
  set -- "-DMFA_VIEW_GROUP=2" "-DMFA_VIEW_GROUP=4" "-DMFA_VIEW_GROUP=8" "-DMFA_VIEW_GROUP=4 -DMFA_VIEW_ORDER=2" "-DMFA_VIEW_GROUP=16 -DMFA_VIEW_ORDER=2"
fi
for f in "$@"; do run "$f"; done
python -m paper_2204_11762_b200.build > /dev/null 2>&1
