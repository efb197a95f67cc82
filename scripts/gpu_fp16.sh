set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -p no:cacheprovider -k "fp16 or config1 or mixed20" > gpurun_out/pytest_fp16.txt 2>&1; tail -3 gpurun_out/pytest_fp16.txt
timeout 1800 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --lookup-fp16 > gpurun_out/bench_fp16.txt 2>&1
tail -1 gpurun_out/bench_fp16.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fp32', d['value'], d['extra']['lookup_ms_per_step']); print('fp16', d['fp16_lookup_mode'])"
