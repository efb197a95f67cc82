set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -p no:cacheprovider -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --series 4096 --steps 2 --warmup 1 --cpu-seconds 2 --no-e2e > gpurun_out/bench_small.txt 2>&1; tail -2 gpurun_out/bench_small.txt
bash scripts/ncu_one.sh prof_knn knn_sweep 1 python scripts/prof_xmap.py 512 1450
bash scripts/ncu_one.sh prof_lookup lookup_xmap 0 python scripts/prof_xmap.py 1024 1450
