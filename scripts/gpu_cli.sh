set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 900 python -m paper_2105_12301_b200 --bench knn --length 10000 --erange 1:20 --fused --output gpurun_out/bench_knn_sweep_L10000.csv; tail -4 gpurun_out/bench_knn_sweep_L10000.csv
timeout 900 python -m paper_2105_12301_b200 --bench lookup --length 10000 --count 1000 --erange 1:20 --output gpurun_out/bench_lookup_sweep_L10000.csv; tail -3 gpurun_out/bench_lookup_sweep_L10000.csv
