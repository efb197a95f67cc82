set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -p no:cacheprovider -k "ccm or convergence" > gpurun_out/pytest_ccm.txt 2>&1; tail -3 gpurun_out/pytest_ccm.txt
timeout 1700 python scripts/bench_ccm.py 256 100 2>&1 | tail -1
