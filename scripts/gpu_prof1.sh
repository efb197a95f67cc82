set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n512.csv python scripts/prof_xmap.py 512 1450 > gpurun_out/prof_run.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"knn_sweep|lookup_xmap" -c 3 -o gpurun_out/prof_v1 python scripts/prof_xmap.py 512 1450 > gpurun_out/prof_full.txt 2>&1
tail -5 gpurun_out/prof_full.txt
