# A/B of two libcmb200 builds on a config-4-shaped shard (T = 10,000, non-resident lookup)
mkdir -p gpurun_out
for i in 1 2; do
for lib in paper_2105_12301_b200/libcmb200_prev.so paper_2105_12301_b200/libcmb200.so; do
  CMB_LIB=$PWD/$lib timeout 900 python scripts/config4_shard.py ${C4_N:-8192} 10000 8 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['shard_s'],3), round(d['tables_s'],3), round(d['lookup_s'],3), d['oracle_check']['max_abs_rho_diff'])"
done; done
