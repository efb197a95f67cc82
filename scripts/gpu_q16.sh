# 16-bit fixed-point target lookup (CMB_LOOKUP_FP16=2): parity tests + full-size timing and deviation
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -p no:cacheprovider -k "fp16 or q16" > gpurun_out/pytest_q16.txt 2>&1; tail -3 gpurun_out/pytest_q16.txt
timeout 1800 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --lookup-fp16 ${Q16_MODES:-2} > gpurun_out/bench_q16.txt 2>&1
tail -1 gpurun_out/bench_q16.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fp32', d['value'], d['extra']['lookup_ms_per_step']); print(json.dumps(d['fp16_lookup_mode'], indent=1))"
