mkdir -p gpurun_out/l2
for alt in "" "--no-alternate"; do
  tag=${alt:-alt}
  ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum -k regex:step_kernel_dyn -s 30 -c 6 --csv python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-e2e $alt > gpurun_out/l2/$tag.csv 2> gpurun_out/l2/$tag.err
done
