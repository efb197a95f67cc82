set -x
bash scripts/ncu_one.sh prof_restricted restricted_records 2 python scripts/bench_ccm.py 32 5
python scripts/ncu_summary.py gpurun_out/prof_restricted 30 | head -40
python scripts/ncu_breakdown.py gpurun_out/prof_restricted 1 8 | head -14
