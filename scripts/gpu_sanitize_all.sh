# memcheck, racecheck, synccheck, initcheck over every device path (scripts/sanitize_small.py)
mkdir -p gpurun_out
bash scripts/gpu_sanitize.sh
bash scripts/gpu_sanitize2.sh
