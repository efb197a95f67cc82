# parity suite + full bench after the shifted-moment lookup change
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 1200 python bench.py > gpurun_out/bench_full.txt 2>&1
tail -1 gpurun_out/bench_full.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('full', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['roofline_smem']['frac'], d['extra']['tables_ms_per_step'], d['extra']['lookup_ms_per_step'], d['clocks'])"
