# two ranks sharing one GPU (gloo): bench --gpus 2 with the N > 1 e2e leg
mkdir -p gpurun_out
export CMB_DIST_BACKEND=gloo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus 2 --series 4096 --steps 2 --warmup 3 > gpurun_out/bench_2rank.txt 2>&1; tail -1 gpurun_out/bench_2rank.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e'], d['n_gpus'])"
tail -5 gpurun_out/bench_2rank.txt | cut -c1-300
