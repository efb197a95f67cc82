set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_io.py -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_io.txt 2>&1; tail -3 gpurun_out/pytest_io.txt
timeout 900 python scripts/bench_io.py 16384 > gpurun_out/bench_io.txt 2>&1; tail -2 gpurun_out/bench_io.txt
