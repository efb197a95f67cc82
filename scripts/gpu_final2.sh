# end-of-session evidence for the committed build: parity + smoke, default bench, reference arm, q16 side mode
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_state.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 1800 python bench.py > gpurun_out/bench_full.txt 2>&1; tail -1 gpurun_out/bench_full.txt | cut -c1-300
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 --cpu-seconds 20 > gpurun_out/bench_ref.txt 2>&1; tail -1 gpurun_out/bench_ref.txt | cut -c1-300
timeout 1800 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --lookup-fp16 2 > gpurun_out/bench_q16.txt 2>&1; tail -1 gpurun_out/bench_q16.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(d['fp16_lookup_mode']))"
