# A/B of two libcmb200 builds on the long-series (non-resident) lookup: N = 1,024, T = 10,000
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 800 -p no:cacheprovider 2>&1 | tail -2
for i in 1 2; do
for lib in paper_2105_12301_b200/libcmb200_prev.so paper_2105_12301_b200/libcmb200.so; do
  CMB_LIB=$PWD/$lib timeout 900 python bench.py --series 1024 --length 10000 --steps 2 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],1), round(d['extra']['tables_ms_per_step'],1), round(d['extra']['lookup_ms_per_step'],1), d['clocks']['sm_mhz'])"
done; done
