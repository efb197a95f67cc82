# ncu --set full capture of the table sweep (xmap TABLE mode) and the edim sweep at N=2048
set -x
mkdir -p gpurun_out
bash scripts/ncu_one.sh prof_knn_edim knn_sweep 0 python scripts/prof_xmap.py 2048 1450
bash scripts/ncu_one.sh prof_knn_table knn_sweep 1 python scripts/prof_xmap.py 2048 1450
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n2048.csv python scripts/prof_xmap.py 2048 1450 > gpurun_out/launches_n2048.log 2>&1
ls -la gpurun_out
