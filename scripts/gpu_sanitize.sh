set -x
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_small.py > gpurun_out/sanitize_memcheck.txt 2>&1; tail -6 gpurun_out/sanitize_memcheck.txt
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python scripts/sanitize_small.py > gpurun_out/sanitize_racecheck.txt 2>&1; tail -6 gpurun_out/sanitize_racecheck.txt
