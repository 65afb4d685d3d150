#!/bin/bash
# One GPU session's evidence (run on the box: bash tools/gpu_round.sh TAG):
# tests, smoke, bench (both arms + the C3-share scaling record), every BASELINE
# config, the Exp 1/3 analogues, the smoke launch list under ncu, and ncu
# captures of the step kernel (C1), the shared-memory grid (C0) and the
# persistent cluster kernel (C4).
TAG=${1:-round}
O=gpurun_out/$TAG
mkdir -p "$O"
nvidia-smi > "$O/smi.txt" 2>&1
run() { local name=$1; shift; timeout "$@"; echo "$name rc=$?" >> "$O/rc.txt"; }
run smoke 300 python -c "import __graft_entry__ as g; g.smoke()" > "$O/smoke.log" 2>&1
run pytest 1500 python -m pytest tests -m gpu -q > "$O/pytest_gpu.log" 2>&1
run bench 400 python bench.py > "$O/bench.json" 2> "$O/bench.err"
run bench_ref 400 python bench.py --impl reference > "$O/bench_ref.json" 2> "$O/bench_ref.err"
run bench_scaling 600 python bench.py --scaling --steps 20 > "$O/bench_scaling.json" 2> "$O/bench_scaling.err"
run configs 900 python tools/bench_configs.py --reps 5 > "$O/configs.jsonl" 2> "$O/configs.err"
run exp3_c0 300 python -m paper_2507_20173_b200 gpuexp --exp 3 --fish 1000000 --steps 100 --reps 3 --out "$O/gpuexp3_c0.csv" 2> "$O/gpuexp3_c0.err"
run exp3_c1 300 python -m paper_2507_20173_b200 gpuexp --exp 3 --fish 10000000 --steps 20 --reps 3 --out "$O/gpuexp3_c1.csv" 2> "$O/gpuexp3_c1.err"
run exp3_c4 300 python -m paper_2507_20173_b200 gpuexp --exp 3 --fish 4096 --steps 20000 --reps 3 --out "$O/gpuexp3_c4.csv" 2> "$O/gpuexp3_c4.err"
run exp1_c1 300 python -m paper_2507_20173_b200 gpuexp --exp 1 --fish 10000000 --steps 20 --reps 3 --out "$O/gpuexp1_c1.csv" 2> "$O/gpuexp1_c1.err"
run ncu_smoke 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$O/smoke_launches.csv" python -c "import __graft_entry__ as g; g.smoke()" > "$O/smoke_ncu.log" 2>&1
run capture 1200 bash tools/capture_profiles.sh "$TAG" regex:step_kernel_dyn
for K in "c0 regex:sgrid_kernel 1e6 100" "c4 regex:cluster_kernel 4096 20000"; do
  set -- $K
  run "ncu_$1" 600 ncu --set full --clock-control none --import-source on -k "$2" -c 1 -f -o "$O/$1" python tools/one_run.py "$3" "$4" > "$O/ncu_$1.log" 2>&1
  ncu -i "$O/$1.ncu-rep" --page raw --csv > "$O/$1_raw.csv" 2>/dev/null
  ncu -i "$O/$1.ncu-rep" --page details --csv > "$O/$1_details.csv" 2>/dev/null
  ncu -i "$O/$1.ncu-rep" --page source --csv --print-source sass > "$O/$1_source.csv" 2>/dev/null
done
cat "$O/rc.txt"
