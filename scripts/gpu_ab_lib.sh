# A/B two builds of libcmb200 (CMB_LIB) on the full bench, interleaved
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 500 -p no:cacheprovider 2>&1 | tail -2
for i in 1 2; do
for lib in paper_2105_12301_b200/libcmb200_prev.so paper_2105_12301_b200/libcmb200.so; do
  CMB_LIB=$PWD/$lib timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],1), round(d['extra']['tables_ms_per_step'],1), round(d['extra']['lookup_ms_per_step'],1), d['clocks']['sm_mhz'])"
done; done
