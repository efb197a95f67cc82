# parity tests + small A/B bench of the kNN sweep (v5 tile kernel vs CMB_KNN_V4=1)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu.txt 2>&1; tail -15 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 600 python bench.py --series ${N:-4096} --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_v5.txt 2>&1; tail -1 gpurun_out/bench_v5.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('v5', d['ms_per_step'], d['extra'])"
CMB_KNN_V4=1 timeout 600 python bench.py --series ${N:-4096} --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_v4.txt 2>&1; tail -1 gpurun_out/bench_v4.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('v4', d['ms_per_step'], d['extra'])"
