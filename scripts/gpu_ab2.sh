# A/B of the kNN table build: tile kernel vs v4, N=4096 and full size (no e2e / cpu legs)
set -x
mkdir -p gpurun_out
for impl in tile v4; do
  if [ $impl = tile ]; then unset CMB_KNN_V4; else export CMB_KNN_V4=1; fi
  timeout 600 python bench.py --series 4096 --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_${impl}_4096.txt 2>&1
  tail -1 gpurun_out/bench_${impl}_4096.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$impl 4096', d['ms_per_step'], d['extra']['tables_ms_per_step'], d['extra']['edim_seconds'])"
done
unset CMB_KNN_V4
timeout 1200 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_tile_full.txt 2>&1
tail -1 gpurun_out/bench_tile_full.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tile full', d['ms_per_step'], d['value'], d['extra'])"
