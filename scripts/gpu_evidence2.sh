set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_full.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/launches_full.log 2>&1
tail -1 gpurun_out/launches_full.log | cut -c1-200
bash scripts/ncu_one.sh prof_lookup_t10k lookup_xmap 0 python bench.py --series 1024 --length 10000 --steps 1 --warmup 0 --no-e2e --no-cpu
python scripts/ncu_summary.py gpurun_out/prof_lookup_t10k 30 | head -36
bash scripts/ncu_one.sh prof_tile_t10k knn_tile 1 python bench.py --series 1024 --length 10000 --steps 1 --warmup 0 --no-e2e --no-cpu
python scripts/ncu_summary.py gpurun_out/prof_tile_t10k 5 | head -26
