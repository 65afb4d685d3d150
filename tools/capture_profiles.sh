#!/bin/bash
# The round's profiling evidence, on the GPU box (one GPU):
#   bash tools/capture_profiles.sh TAG [KERNEL_REGEX] [EXTRA_BENCH_ARGS]
# 1. bench.py (default run) -> bench.json          (must exit 0 before any ncu pass)
# 2. launch list of bench.py --steps 20 --warmup 3 (gpu__time_duration.sum, --clock-control none)
# 3. ncu --set full of one step-kernel launch (cold cache), exported as details / raw / source CSV
# 4. DRAM bytes of six consecutive launches with the L2 state carried (--cache-control none)
TAG=${1:?tag}
KRE=${2:-regex:step_kernel}
X=${3:-}
OUT=gpurun_out/prof_$TAG
mkdir -p "$OUT"
python bench.py $X > "$OUT/bench.json" 2> "$OUT/bench.err" || { echo "bench failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file "$OUT/launches.csv" \
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $X > "$OUT/ncu_launches.log" 2>&1
ncu --set full --clock-control none --import-source on -k "$KRE" -s 10 -c 1 -f -o "$OUT/step" \
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $X > "$OUT/ncu_full.log" 2>&1
ncu -i "$OUT/step.ncu-rep" --page details --csv > "$OUT/step_details.csv" 2>/dev/null
ncu -i "$OUT/step.ncu-rep" --page raw --csv > "$OUT/step_raw.csv" 2>/dev/null
ncu -i "$OUT/step.ncu-rep" --page source --csv --print-source sass > "$OUT/step_source.csv" 2>/dev/null
ncu --cache-control none --clock-control none \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
  -k "$KRE" -s 30 -c 6 --csv python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-e2e $X \
  > "$OUT/warm_l2.csv" 2> "$OUT/warm_l2.err"
ls -la "$OUT"
