#!/bin/bash
# DRAM bytes per step-kernel launch with the L2 state carried between launches
# (ncu --cache-control none), for each library variant named on the command line.
#   bash tools/l2_reuse_probe.sh default keep30 ...   (on the GPU box)
mkdir -p gpurun_out
for v in "$@"; do
  FSB_L2_VERBOSE=1 FSB_LIB=build/variants/libfsb_$v.so ncu --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    -k regex:step_kernel -s 30 -c 6 --csv python tools/bench_configs.py --only C1 --reps 1 \
    > gpurun_out/l2probe_$v.csv 2> gpurun_out/l2probe_$v.err
done
