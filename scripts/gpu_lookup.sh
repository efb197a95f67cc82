# lookup iteration: GPU tests, full-size step timing (no e2e / cpu legs)
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x > gpurun_out/pytest_gpu.txt 2>&1; tail -4 gpurun_out/pytest_gpu.txt
timeout 1500 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_full_nocpu.txt 2>&1
tail -1 gpurun_out/bench_full_nocpu.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('full', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline_smem']['frac'], d['extra'])"
bash scripts/ncu_one.sh prof_lookup_full lookup_xmap 3 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu
python scripts/ncu_summary.py gpurun_out/prof_lookup_full 5 | head -34
