# round evidence: parity + smoke, default bench (e2e + cpu baseline), launch list, ncu of both hot kernels
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_state.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 1800 python bench.py > gpurun_out/bench_full.txt 2>&1; tail -1 gpurun_out/bench_full.txt | cut -c1-400
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_full.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/launches_full.log 2>&1
bash scripts/ncu_one.sh prof_tile_full knn_tile 12 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu
bash scripts/ncu_one.sh prof_tile_table knn_tile 1 python scripts/prof_xmap.py 1024 1450
ls gpurun_out
