# iteration check: GPU tests, small bench, per-kernel ncu captures
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu.txt 2>&1
tail -15 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --n 4096 --steps 2 --warmup 1 --cpu-seconds 3 --no-e2e > gpurun_out/bench_small.txt 2>&1; tail -3 gpurun_out/bench_small.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n1024.csv python scripts/prof_xmap.py 1024 1450 > gpurun_out/prof_run.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:knn_sweep -s 1 -c 1 -o gpurun_out/prof_knn python scripts/prof_xmap.py 512 1450 > gpurun_out/prof_knn.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lookup_xmap -c 1 -o gpurun_out/prof_lookup python scripts/prof_xmap.py 1024 1450 > gpurun_out/prof_lookup.txt 2>&1
tail -3 gpurun_out/prof_knn.txt gpurun_out/prof_lookup.txt
