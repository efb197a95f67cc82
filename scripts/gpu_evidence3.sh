# round evidence for the current build: tests, smoke, bench (both arms), launch list, ncu captures
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_state.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 1800 python bench.py > gpurun_out/bench_full.txt 2>&1
tail -1 gpurun_out/bench_full.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('full', d['value'], d['ms_per_step'], d['e2e']['value'], d['cpu_baseline']['value'], d['roofline']['frac'], d['roofline_smem']['frac'], d['extra']['tables_ms_per_step'], d['extra']['lookup_ms_per_step'], d['clocks'])"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 --cpu-seconds 20 > gpurun_out/bench_ref.txt 2>&1; tail -1 gpurun_out/bench_ref.txt | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_full.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/launches_full.log 2>&1
bash scripts/ncu_one.sh prof_tile_full knn_tile 12 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu
python scripts/ncu_summary.py gpurun_out/prof_tile_full 5 2>/dev/null | head -40
bash scripts/ncu_one.sh prof_lookup_full lookup_xmap 4 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu
python scripts/ncu_summary.py gpurun_out/prof_lookup_full 5 2>/dev/null | head -40
rm -f gpurun_out/*.ncu-rep
