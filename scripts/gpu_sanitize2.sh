set -x
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool synccheck --num-cuda-barriers 64 --print-limit 20 python scripts/sanitize_small.py > gpurun_out/sanitize_synccheck.txt 2>&1; tail -3 gpurun_out/sanitize_synccheck.txt
timeout 1500 compute-sanitizer --tool initcheck --print-limit 20 python scripts/sanitize_small.py > gpurun_out/sanitize_initcheck.txt 2>&1; tail -12 gpurun_out/sanitize_initcheck.txt
