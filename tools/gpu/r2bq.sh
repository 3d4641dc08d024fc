# round 2, call bq: the large-K full-run test on every path
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "full_run_large_k" > gpurun_out/r2bq_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2bq_tests.txt
