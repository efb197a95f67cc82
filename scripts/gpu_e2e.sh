# GPU tests + default bench (e2e + cpu baseline legs)
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 1800 python bench.py > gpurun_out/bench_full.txt 2>&1
tail -1 gpurun_out/bench_full.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('full', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'], d['e2e']['ms_per_step'], 'cpu', d['cpu_baseline']['value'], d['clocks'])"
