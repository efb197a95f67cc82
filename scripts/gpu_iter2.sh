# iteration: GPU tests (incl. tile-vs-v4 A/B), N=4096 timing, ncu breakdown of the tile kernel
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x > gpurun_out/pytest_gpu.txt 2>&1; tail -4 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --series 4096 --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_tile_4096.txt 2>&1
tail -1 gpurun_out/bench_tile_4096.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tile 4096', d['ms_per_step'], d['extra']['tables_ms_per_step'], d['extra']['edim_seconds'], d['extra']['exact_fallback_rows'])"
bash scripts/ncu_one.sh prof_tile_table knn_tile 1 python scripts/prof_xmap.py 1024 1450
python scripts/ncu_breakdown.py gpurun_out/prof_tile_table 29501440 16
