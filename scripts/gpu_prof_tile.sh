# --set full capture of the tile kNN kernel in TABLE mode at T = 1,450 (N = 2,048 libraries)
mkdir -p gpurun_out
python scripts/prof_xmap.py 2048 1450
bash scripts/ncu_one.sh prof_tile_t1450 knn_tile 1 python scripts/prof_xmap.py 2048 1450
python scripts/ncu_summary.py gpurun_out/prof_tile_t1450 5 | head -30
python scripts/ncu_breakdown.py gpurun_out/prof_tile_t1450 $((2048*1440*20)) 30
