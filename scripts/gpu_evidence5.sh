# headline evidence after the interleaved-row tile kernel: bench (e2e + cpu baseline), reference arm,
# config-2 edim, launch list, smoke
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 1800 python bench.py > gpurun_out/bench_full.txt 2>&1
tail -1 gpurun_out/bench_full.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('full', d['value'], d['ms_per_step'], d['e2e']['value'], d['cpu_baseline']['value'], d['roofline']['frac'], d['roofline_smem']['frac'], d['extra']['tables_ms_per_step'], d['extra']['lookup_ms_per_step'], d['extra']['edim_seconds'], d['clocks'])"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 --cpu-seconds 20 > gpurun_out/bench_ref.txt 2>&1; tail -1 gpurun_out/bench_ref.txt | cut -c1-200
timeout 600 python scripts/edim_cfg2.py > gpurun_out/edim_cfg2.txt 2>&1; tail -1 gpurun_out/edim_cfg2.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_full.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/launches_full.log 2>&1
