set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
(nproc; lscpu | head -20) > gpurun_out/host.txt 2>&1
python -c "import torch;p=torch.cuda.get_device_properties(0);print(p, p.multi_processor_count, p.L2_cache_size)" >> gpurun_out/host.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
tail -40 gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke.txt 2>&1; tail -5 gpurun_out/smoke.txt
timeout 600 python bench.py --series 4096 --steps 2 --warmup 1 --cpu-seconds 5 > gpurun_out/bench_small.txt 2>&1; tail -5 gpurun_out/bench_small.txt
timeout 1200 python bench.py --cpu-seconds 10 > gpurun_out/bench_full.txt 2>&1; tail -5 gpurun_out/bench_full.txt
