set -x
mkdir -p gpurun_out
timeout 900 python bench.py --series 1024 --length 10000 --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_t10k.txt 2>&1; tail -1 gpurun_out/bench_t10k.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('t10k', d['value'], d['ms_per_step'], d['extra']['tables_ms_per_step'], d['extra']['lookup_ms_per_step'])"
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
