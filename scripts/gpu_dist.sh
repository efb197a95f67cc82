# multi-rank functional runs sharing one GPU (gloo): sharded xmap == single process; bench --gpus 2
set -x
mkdir -p gpurun_out
export CMB_DIST_BACKEND=gloo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 scripts/dist_check.py 300 1450 > gpurun_out/dist_check.txt 2>&1; tail -3 gpurun_out/dist_check.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus 2 --series 2048 --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_2rank.txt 2>&1; tail -2 gpurun_out/bench_2rank.txt | cut -c1-300
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29563 bench.py --impl reference --gpus 2 --series 2048 --steps 1 --warmup 0 --cpu-seconds 4 > gpurun_out/bench_ref_2rank.txt 2>&1; tail -2 gpurun_out/bench_ref_2rank.txt | cut -c1-300
