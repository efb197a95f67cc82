# refresh the launch list and the lookup --set full capture for the current build
set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_full.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/launches_full.log 2>&1
bash scripts/ncu_one.sh prof_lookup_full lookup_xmap 4 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu
python scripts/ncu_summary.py gpurun_out/prof_lookup_full 5 2>/dev/null | head -40
rm -f gpurun_out/*.ncu-rep
