# iteration check: GPU tests, small bench, per-kernel ncu captures
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu.txt 2>&1
tail -15 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --series 4096 --steps 2 --warmup 1 --cpu-seconds 3 --no-e2e > gpurun_out/bench_small.txt 2>&1; tail -3 gpurun_out/bench_small.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n1024.csv python scripts/prof_xmap.py 1024 1450 > gpurun_out/prof_run.txt 2>&1
bash scripts/ncu_one.sh prof_knn knn_sweep 1 python scripts/prof_xmap.py 512 1450
bash scripts/ncu_one.sh prof_lookup lookup_xmap 0 python scripts/prof_xmap.py 1024 1450
ls -la gpurun_out
