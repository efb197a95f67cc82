# parity suite on the new build, then A/B of two builds of libcmb200 (CMB_LIB) on the full bench, interleaved
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 800 -p no:cacheprovider 2>&1 | tail -3
for i in 1 2; do
for lib in paper_2105_12301_b200/libcmb200_prev.so paper_2105_12301_b200/libcmb200.so; do
  CMB_LIB=$PWD/$lib timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],1), round(d['extra']['tables_ms_per_step'],1), round(d['extra']['lookup_ms_per_step'],1), d['clocks']['sm_mhz'])"
done; done
