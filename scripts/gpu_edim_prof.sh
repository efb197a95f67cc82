set -x
mkdir -p gpurun_out
bash scripts/ncu_one.sh prof_tile_edim knn_tile 0 python scripts/prof_xmap.py 1024 1450
python scripts/ncu_breakdown.py gpurun_out/prof_tile_edim 29480960 16
python scripts/ncu_summary.py gpurun_out/prof_tile_edim 5 | head -16
