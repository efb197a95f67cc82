# long-series paths: config 2 (edim 1,024 x 10,000) tile vs v4, config-4-shaped xmap slice
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 900 python scripts/edim_cfg2.py 256 10000 > gpurun_out/cfg2_tile_256.txt 2>&1; cat gpurun_out/cfg2_tile_256.txt
CMB_KNN_V4=1 timeout 900 python scripts/edim_cfg2.py 256 10000 > gpurun_out/cfg2_v4_256.txt 2>&1; cat gpurun_out/cfg2_v4_256.txt
timeout 900 python bench.py --series 1024 --length 10000 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_t10k.txt 2>&1; tail -1 gpurun_out/bench_t10k.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('t10k', d['value'], d['ms_per_step'], d['extra'])"
