# tile-kernel iteration: parity (CMB_KNN_TILE=1), selection stats, A/B timing at N=4096, ncu of the tile kernel
set -x
mkdir -p gpurun_out
unset CMB_KNN_V4
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu.txt 2>&1; tail -5 gpurun_out/pytest_gpu.txt
python scripts/knn_stats2.py 1024 > gpurun_out/knn_stats.txt 2>&1; cat gpurun_out/knn_stats.txt
timeout 600 python bench.py --series 4096 --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_tile.txt 2>&1; tail -1 gpurun_out/bench_tile.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tile', d['ms_per_step'], d['extra'])"
bash scripts/ncu_one.sh prof_tile_table knn_tile 1 python scripts/prof_xmap.py 1024 1450
python scripts/ncu_summary.py gpurun_out/prof_tile_table 30 | head -24
